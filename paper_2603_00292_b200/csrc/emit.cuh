// emit.cuh -- K4+K5: fused Karras emission + bottom-up refit (included by lbvh.cu
// inside its anonymous namespace; uses load_tri / tri_box / adj_delta from there).
//
// One thread per leaf climbs the tree (Apetrei 2014's agglomerative scheme): a
// node covering keys [l, r] is the LEFT child of its parent iff
// delta(r, r+1) > delta(l-1, l) (no ties exist for index-augmented keys).
// Siblings meet at the parent's split slot gamma: the first arrival publishes
// its box and leaves, the second builds the parent.  Karras's numbering
// (internal 0..n-2, root 0) is recovered exactly: a left child is numbered by
// its right end, a right child by its left end, so child / parent arrays equal
// the split-search construction bit for bit (oracle orc_lbvh_karras/refit).
//
// Phase A (per block of EMIT_T leaves [B, E)): pairs whose sibling starts
// inside the block meet in SHARED memory (ATOMS exchange, delta read from a
// per-block smem table) -- no global latency on the chain.  A node whose
// sibling starts outside the block is deferred.  Phase B (after one barrier):
// deferred nodes and smem slots that saw a single arrival (the sibling
// extends past the block) climb through the global slots: a release exchange
// after st.cg of the box, the sibling's box read with ld.cg (no device-scope
// acquire fence, which would invalidate the whole L1 on every rendezvous).
//
// node layout (Aila-Laine): n0 = (L.lo.x, L.hi.x, L.lo.y, L.hi.y)
//                           n1 = (R.lo.x, R.hi.x, R.lo.y, R.hi.y)
//                           n2 = (L.lo.z, L.hi.z, R.lo.z, R.hi.z)
//                           n3 = (left id, right id, height, 0)   id < 0: ~leaf
#pragma once

struct EmitNode {
    int l, r, h, dl, dr;
    int g;                 // split position this node was created at (BVH4 index); -1 for a leaf
    float lo[3], hi[3];
};

// BVH4 view, indexed by binary SPLIT position: the BVH4 node of the binary node
// with split g holds that node's up-to-4 grandchildren (a leaf child stays a
// leaf).  Each binary node knows its parent's split as soon as it exists (the
// side test), so it writes its own half -- slots 2*side, 2*side+1 = its two
// children, or itself if a leaf -- with no cross-thread reads.  Layout: 4 slots
// of 2 float4 = (lo.xyz, child id), (hi.xyz, 0); the child id is the split
// position of an internal grandchild or ~leaf.  A half is 64 contiguous bytes.
#ifndef RT_STG256
#define RT_STG256 1
#endif
// 1: also write the Karras child ids per internal node (8 scattered bytes each); 0: the
// download derives them from the BVH4 halves (see bvh4_write_half)
#ifndef RT_EMIT_CHILD
#define RT_EMIT_CHILD 0
#endif
// The half also records its writer's own BVH4 id (`self`: the writer's split, or ~leaf)
// in the spare .w of its first hi vector: with it rt_bvh_download rebuilds the binary
// topology (each node's children and Karras numbers) from the BVH4 view alone, so the
// build writes no separate child array.
__device__ __forceinline__ void bvh4_write_half(float4* __restrict__ bvh4, int pgamma, int side, const float a_lo[3],
                                                const float a_hi[3], int a_id, const float b_lo[3],
                                                const float b_hi[3], int b_id, int self) {
    float4* q = bvh4 + 8 * (int64_t)pgamma + 4 * side;
#if RT_STG256
    // two 256-bit stores (sm_100 STG.E.256) per 64-B half; the half is 64-B aligned
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(q), "f"(a_lo[0]), "f"(a_lo[1]),
                 "f"(a_lo[2]), "f"(__int_as_float(a_id)), "f"(a_hi[0]), "f"(a_hi[1]), "f"(a_hi[2]),
                 "f"(__int_as_float(self))
                 : "memory");
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(q + 2), "f"(b_lo[0]), "f"(b_lo[1]),
                 "f"(b_lo[2]), "f"(__int_as_float(b_id)), "f"(b_hi[0]), "f"(b_hi[1]), "f"(b_hi[2]), "f"(0.0f)
                 : "memory");
#else
    q[0] = make_float4(a_lo[0], a_lo[1], a_lo[2], __int_as_float(a_id));
    q[1] = make_float4(a_hi[0], a_hi[1], a_hi[2], __int_as_float(self));
    q[2] = make_float4(b_lo[0], b_lo[1], b_lo[2], __int_as_float(b_id));
    q[3] = make_float4(b_hi[0], b_hi[1], b_hi[2], 0.0f);
#endif
}

// a leaf writes itself + an empty slot into its parent's BVH4 node
__device__ __forceinline__ void bvh4_write_leaf(float4* __restrict__ bvh4, const EmitNode& N) {
    const bool left = N.dr > N.dl;
    if (N.dr < 0 && N.dl < 0) return;                // n == 1: no parent
    // empty slot: lo = hi = +inf on every axis.  (lo = +inf, hi = -inf would be an
    // INFINITE box for the min/max slab test, which orders each slab's ends.)
    const float elo[3] = {INFINITY, INFINITY, INFINITY}, ehi[3] = {INFINITY, INFINITY, INFINITY};
    bvh4_write_half(bvh4, left ? N.r : N.l - 1, left ? 0 : 1, N.lo, N.hi, ~N.l, elo, ehi, ~0, ~N.l);
}

// Emit the parent of N (N is the left child iff `left`) whose sibling brought
// `other` (its far endpoint), box (s0 = lo + height, s1 = hi + its split g);
// pdl / pdr are delta at the parent's boundaries.  N becomes the parent, which
// also writes its half of ITS parent's BVH4 node (or records the BVH4 root).
// Returns true at the root.
__device__ __forceinline__ bool emit_parent(int64_t n, int2* __restrict__ child, float4* __restrict__ nodes, float4* __restrict__ bvh4, EmitNode& N,
                                            bool left, int gamma, int pl, int pr, int pdl, int pdr,
                                            const float4 s0, const float4 s1) {
    const int cl = (pl == gamma) ? ~gamma : gamma;
    const int cr = (pr == gamma + 1) ? ~(gamma + 1) : gamma + 1;
    float llo[3], lhi[3], rlo[3], rhi[3];
    const float so[3] = {s0.x, s0.y, s0.z}, sh[3] = {s1.x, s1.y, s1.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        llo[a] = left ? N.lo[a] : so[a]; lhi[a] = left ? N.hi[a] : sh[a];
        rlo[a] = left ? so[a] : N.lo[a]; rhi[a] = left ? sh[a] : N.hi[a];
    }
    const int hs = __float_as_int(s0.w), gs = __float_as_int(s1.w);
    // BVH4 ids of the two children: split position if internal, ~leaf otherwise
    const int gl = (pl == gamma) ? ~gamma : (left ? N.g : gs);
    const int gr = (pr == gamma + 1) ? ~(gamma + 1) : (left ? gs : N.g);
    const bool root = (pl == 0 && pr == n - 1);
    const bool pleft = pdr > pdl;
#if RT_EMIT_CHILD
    const int P = root ? 0 : (pleft ? pr : pl);
#endif
    N.h = 1 + (N.h > hs ? N.h : hs);
    // Only the topology (child ids, 8 B) and the BVH4 half are written per node: the
    // binary node's child boxes ARE that half, so parent pointers, per-node boxes and
    // heights are derived from child + bvh4 by rt_bvh_download (parity only).  The
    // root alone writes its 64-B record (child boxes, ids, tree height, BVH4 root).
#if RT_EMIT_CHILD
    child[P] = make_int2(cl, cr);
#endif
    if (root) {
        nodes[0] = make_float4(llo[0], lhi[0], llo[1], lhi[1]);
        nodes[1] = make_float4(rlo[0], rhi[0], rlo[1], rhi[1]);
        nodes[2] = make_float4(llo[2], lhi[2], rlo[2], rhi[2]);
        nodes[3] = make_float4(__int_as_float(cl), __int_as_float(cr), __int_as_float(N.h), __int_as_float(gamma));
    } else {
        bvh4_write_half(bvh4, pleft ? pr : pl - 1, pleft ? 0 : 1, llo, lhi, gl, rlo, rhi, gr, gamma);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) { N.lo[a] = sel_min(llo[a], rlo[a]); N.hi[a] = sel_max(lhi[a], rhi[a]); }
    N.l = pl; N.r = pr; N.dl = pdl; N.dr = pdr; N.g = gamma;
    return root;
}

// Global rendezvous without a release fence: a fence.gpu before the exchange would wait
// for every earlier store of the thread (the previous level's node writes) to reach L2,
// on each level of the chain.  Instead the box halves carry validity tags in .w
// (height | (outer delta + 1) << 8 >= 0, split g >= -1; both sides' tags are invalidated
// by the emit kernel's hand-off before this kernel runs), the exchange is relaxed, and
// the second arrival spins on the L2 copy of its sibling's box until both tags are
// valid.  (Records are written and read as single 256-bit accesses of one 32-B sector.)
constexpr int SLOT_INVALID = (int)0x80000000;

#ifndef EMIT_ACQREL
#define EMIT_ACQREL 1
#endif
__device__ __forceinline__ int atom_exch_acq_rel_cta(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.cta.shared::cta.exch.b32 %0, [%1], %2;"
                 : "=r"(old)
                 : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
                 : "memory");
    return old;
}

// A spin on a plain (even asm-volatile ld.global.cg) load is NOT a loop to ptxas: it
// assumes the location cannot change and keeps at most one reload.  The re-reads must be
// strong relaxed loads at GPU scope, which ptxas must re-issue on every iteration.
// A slot record is 32 B (box lo + tag, box hi + split) and moves as ONE 256-bit access.
__device__ __forceinline__ void ld_record_relaxed(const float4* p, float4& a, float4& b) {
    asm volatile("ld.relaxed.gpu.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ void ld_record_cg(const float4* p, float4& a, float4& b) {
    asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ void st_record_cg(float4* p, const float4 a, const float4 b) {
    asm volatile("st.global.cg.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a.x), "f"(a.y), "f"(a.z),
                 "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                 : "memory");
}

template <typename K>
__device__ void climb_global(const K* __restrict__ keys, int64_t n, int2* __restrict__ child,
                             float4* __restrict__ nodes, float4* __restrict__ bvh4, int* slot_range,
                             float4* slot_box, EmitNode N) {
    while (true) {
        const bool left = N.dr > N.dl;
        const int gamma = left ? N.r : N.l - 1;
        const int side = left ? 0 : 1;
        // the box record also carries this node's OUTER boundary delta (the parent's
        // boundary on this side: dl for a left child, dr for a right child), so the
        // second arrival needs no key loads: one L2 round trip per level (the sibling's
        // record is read speculatively alongside the exchange)
        const int outer = (left ? N.dl : N.dr) + 1;
        st_record_cg(slot_box + 4 * gamma + 2 * side,
                     make_float4(N.lo[0], N.lo[1], N.lo[2], __int_as_float(N.h | (outer << 8))),
                     make_float4(N.hi[0], N.hi[1], N.hi[2], __int_as_float(N.g)));
        const float4* sib = slot_box + 4 * gamma + 2 * (1 - side);
        float4 s0, s1;
        ld_record_cg(sib, s0, s1);
        const int other = atomicExch(slot_range + gamma, left ? N.l : N.r);
        if (other < 0) return;                       // sibling subtree not finished
        while (__float_as_int(s0.w) == SLOT_INVALID || __float_as_int(s1.w) == SLOT_INVALID)
            ld_record_relaxed(sib, s0, s1);
        const int pl = left ? N.l : other, pr = left ? other : N.r;
        const int sd = (__float_as_int(s0.w) >> 8) - 1;
        s0.w = __int_as_float(__float_as_int(s0.w) & 0xFF);
        const int pdl = left ? N.dl : sd;
        const int pdr = left ? sd : N.dr;
        if (emit_parent(n, child, nodes, bvh4, N, left, gamma, pl, pr, pdl, pdr, s0, s1)) return;
    }
}

// invalidate both sides' box tags of a global split slot (emit hand-off)
__device__ __forceinline__ void slot_reset(int* slot_range, float4* slot_box, int gamma) {
    slot_range[gamma] = -1;
    int* b = reinterpret_cast<int*>(slot_box + 4 * (int64_t)gamma);
    b[3] = SLOT_INVALID; b[7] = SLOT_INVALID; b[11] = SLOT_INVALID; b[15] = SLOT_INVALID;
}

// n == 1: the BVH4 root (index 0) holds the single leaf; the other slots are empty
__global__ void bvh4_single_leaf_kernel(const float4* __restrict__ nodes, float4* __restrict__ bvh4) {
    const float4 a0 = nodes[0], a2 = nodes[2];
    const float lo[3] = {a0.x, a0.z, a2.x}, hi[3] = {a0.y, a0.w, a2.y};
    const float e[3] = {INFINITY, INFINITY, INFINITY};
    bvh4_write_half(bvh4, 0, 0, lo, hi, ~0, e, e, ~0, ~0);
    bvh4_write_half(bvh4, 0, 1, e, e, ~0, e, e, ~0, ~0);
}

#ifndef EMIT_TILE
#define EMIT_TILE 256   // 128 / 512 measured slower (1M emit 0.125 -> 0.134 / 0.136 ms)
#endif
constexpr int EMIT_T = EMIT_TILE;

#ifndef EMIT_MINB
#define EMIT_MINB 5   // 48 registers: 5 blocks per SM (10M emit 1.14 -> 1.09 ms)
#endif
template <typename K>
__global__ void __launch_bounds__(EMIT_T, EMIT_MINB) lbvh_emit_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ order,
                                                           const float* __restrict__ tris, const uint32_t* __restrict__ mask,
                                                           uint32_t umask,
                                                           int64_t n, int2* __restrict__ child,
                                                           float4* __restrict__ tri_sorted, float4* __restrict__ nodes,
                                                           float4* __restrict__ bvh4, EmitNode* __restrict__ items,
                                                           unsigned int* __restrict__ seg_count,
                                                           int* __restrict__ slot_range, float4* __restrict__ slot_box) {
    __shared__ int s_range[EMIT_T];             // smem split slots (gamma - B); -1 empty, -2 done
    __shared__ int s_delta[EMIT_T + 1];         // delta(B - 1 + k)
    __shared__ float4 s_box[EMIT_T][2][2];      // [slot][side][(lo, h) | (hi, -)]
    __shared__ unsigned s_cnt;                  // finished subtrees handed to the global climb
    const int tid = threadIdx.x;
    const int64_t B = (int64_t)blockIdx.x * EMIT_T;
    const int64_t E = (B + EMIT_T < n) ? B + EMIT_T : n;
    s_range[tid] = -1;
    pdl_wait();                                 // the sorted keys and order
    pdl_trigger();
    s_delta[tid] = adj_delta(keys, n, B - 1 + tid);
    if (tid == 0) {
        s_cnt = 0;
        s_delta[EMIT_T] = adj_delta(keys, n, B - 1 + EMIT_T);
    }
    const int64_t i = B + tid;
    EmitNode N;
    if (i < E) {
        const uint32_t id = order[i];
        float t[9];
        load_tri_gather(tris, id, t);
        tri_box(t, N.lo, N.hi);
        tri_sorted[3 * i + 0] = make_float4(t[0], t[1], t[2], __int_as_float((int)id));
        tri_sorted[3 * i + 1] = make_float4(t[3], t[4], t[5], __uint_as_float(mask ? mask[id] : umask));
        tri_sorted[3 * i + 2] = make_float4(t[6], t[7], t[8], 0.0f);
        N.l = N.r = (int)i;
        N.h = 0;
        N.g = -1;
    }
    __syncthreads();
    if (i < E) {
        N.dl = s_delta[tid];            // delta(i - 1)
        N.dr = s_delta[tid + 1];        // delta(i)
        bvh4_write_leaf(bvh4, N);
        while (true) {
            const bool left = N.dr > N.dl;
            const bool inside = left ? (N.r + 1 < E) : (N.l - 1 >= B);
            if (!inside) {
                // the block's segment of the hand-off list (no global counter)
                items[B + atomicAdd(&s_cnt, 1u)] = N;
                if (N.r < n - 1) slot_reset(slot_range, slot_box, N.r);
                break;
            }
            const int gamma = left ? N.r : N.l - 1;
            const int g = gamma - (int)B, side = left ? 0 : 1;
            s_box[g][side][0] = make_float4(N.lo[0], N.lo[1], N.lo[2], __int_as_float(N.h));
            s_box[g][side][1] = make_float4(N.hi[0], N.hi[1], N.hi[2], __int_as_float(N.g));
#if EMIT_ACQREL
            // release (publishes this side's box) + acquire (sees the sibling's) in the
            // exchange itself instead of two sequentially consistent block fences
            const int other = atom_exch_acq_rel_cta(&s_range[g], left ? N.l : N.r);
            if (other < 0) break;                    // first arrival: pending in smem
#else
            __threadfence_block();
            const int other = atomicExch(&s_range[g], left ? N.l : N.r);
            if (other < 0) break;                    // first arrival: pending in smem
            __threadfence_block();
#endif
            s_range[g] = -2;                         // pair complete
            const int pl = left ? N.l : other, pr = left ? other : N.r;
            // the parent lies inside the block, so its boundary deltas are in smem
            const int pdl = s_delta[pl - (int)B], pdr = s_delta[pr - (int)B + 1];
            if (emit_parent(n, child, nodes, bvh4, N, left, gamma, pl, pr, pdl, pdr, s_box[g][1 - side][0],
                            s_box[g][1 - side][1]))
                break;                               // root (whole tree inside one block)
        }
    }
    __syncthreads();
    // hand-off to phase B: smem slot `tid` left with a single arrival (its sibling
    // extends past the block) -> this block's segment items[B, B + count)
    if (tid < EMIT_T - 1 && B + tid + 1 < E && s_range[tid] >= 0) {
        const int endpoint = s_range[tid];
        const int gamma = (int)B + tid;
        const bool left = endpoint <= gamma;         // left child: [endpoint, gamma]; right: [gamma+1, endpoint]
        const float4 lo4 = s_box[tid][left ? 0 : 1][0], hi4 = s_box[tid][left ? 0 : 1][1];
        EmitNode M;
        M.l = left ? endpoint : gamma + 1;
        M.r = left ? gamma : endpoint;
        M.h = __float_as_int(lo4.w);
        M.g = __float_as_int(hi4.w);
        M.lo[0] = lo4.x; M.lo[1] = lo4.y; M.lo[2] = lo4.z;
        M.hi[0] = hi4.x; M.hi[1] = hi4.y; M.hi[2] = hi4.z;
        M.dl = s_delta[M.l - (int)B];
        M.dr = s_delta[M.r - (int)B + 1];
        items[B + atomicAdd(&s_cnt, 1u)] = M;
        if (M.r < n - 1) slot_reset(slot_range, slot_box, M.r);   // the global climb's slots: item right ends
    }
    __syncthreads();
    if (tid == 0) seg_count[blockIdx.x] = s_cnt;
}

// Phase B as its own kernel: the few boundary-crossing nodes of all
// blocks (typically ~n/30) climb through the global split slots.  Keeping these
// long, mostly single-lane chains out of kernel A lets its blocks retire at once
// instead of holding an SM slot for the whole chain.  Items come in per-block
// segments items[b * EMIT_T, b * EMIT_T + seg_count[b]), one warp per segment.
template <typename K>
__global__ void __launch_bounds__(128) lbvh_emit_global_kernel(const K* __restrict__ keys, int64_t n,
                                                              int2* __restrict__ child,
                                                              float4* __restrict__ nodes, float4* __restrict__ bvh4,
                                                              int* slot_range, float4* slot_box,
                                                              const EmitNode* __restrict__ items,
                                                              const unsigned int* __restrict__ seg_count,
                                                              int64_t n_blocks, uint4* __restrict__ scratch,
                                                              int64_t scratch_n16) {
    // one warp per segment, so every item climbs concurrently (no thread takes two)
    pdl_wait();                                 // the emit kernel's items and slot resets
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t seg = gt >> 5;
    if (seg < n_blocks) {
        const unsigned cnt = __ldg(seg_count + seg);
        for (unsigned j = threadIdx.x & 31; j < cnt; j += 32)
            climb_global(keys, n, child, nodes, bvh4, slot_range, slot_box, items[seg * EMIT_T + j]);
    }
    // the sort scratch (digit histograms, tile counters, bounds accumulators, look-back
    // status) is dead now: zero it for the next build here, off the climb's critical path,
    // instead of a memset ahead of every build
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = gt; k < scratch_n16; k += stride) scratch[k] = make_uint4(0u, 0u, 0u, 0u);
}
