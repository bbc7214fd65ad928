// lbvh.cu -- GPU LBVH build for sm_100a (replaces the reference's top-down
// binned-SAH _build_bvh, accel.py:68-187, with Karras 2012).
//
//   K1 lbvh_bounds     fp32 centroid bounds (block reduce + one orderable-uint
//                      atomic per block and axis)
//   K2 lbvh_morton     30-bit (10b/axis) or 63-bit (21b/axis) keys, no FMA
//   K3 onesweep        LSD radix sort, one histogram pass for all digits (fused
//                      into K2) + one kernel per digit with decoupled look-back
//                      and warp ranking; stable.  30-bit keys: 3 passes of
//                      10-bit digits; 63-bit keys: 8 passes of 8-bit digits
//   K4+K5 lbvh_emit    fused Karras emission + refit in one bottom-up pass
//                      (index fallback for equal keys, parent pointers, leaf
//                      gather into leaf order, 64-B BVH2 nodes with both child
//                      boxes in the parent + subtree height)
//
// The choices are the frozen ones of SURVEY.md 8(c); oracle/rt_oracle.c Part B
// restates them on the CPU and tests/test_gpu_lbvh.py checks bit equality.
#include <cub/block/block_scan.cuh>
#include <cuda/atomic>
#include <utility>

#include "rt_common.cuh"

namespace {

// Programmatic dependent launch between the build's kernels: each kernel after K1 is
// launched with programmatic stream serialization and waits (griddepcontrol.wait) for its
// predecessor's completion and memory flush before reading the predecessor's outputs, so
// the launch itself overlaps the predecessor's drain (1M build 0.2155 -> 0.1995 ms, 63-bit
// 0.296 -> 0.273 ms, 10M 1.587 -> 1.573 ms).  Explicit early triggers
// (griddepcontrol.launch_dependents, RT_PDL_TRIG) are slower: the waiting dependents take
// SM slots from the multi-wave predecessors (10M 1.57 -> 2.25 ms).  A trigger, if enabled,
// must follow the wait: triggering before it lets grids chain ahead of a still-running
// pass, whose read-only cached lines of the ping-pong key buffers then go stale.
#ifndef RT_PDL
#define RT_PDL 1
#endif
#ifndef RT_PDL_TRIG
#define RT_PDL_TRIG 0
#endif
__device__ __forceinline__ void pdl_trigger() {
#if RT_PDL && RT_PDL_TRIG
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if RT_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_smem(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = RT_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = RT_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

constexpr int SORT_THREADS = 256;   // == RADIX
#ifndef SORT_ITEMS32
#define SORT_ITEMS32 10      // 8 / 9 / 10 with 4 blocks per SM: 10M 0.422 / 0.402 / 0.391 ms
#endif
#ifndef SORT_ITEMS64
#define SORT_ITEMS64 8
#endif
#ifndef SORT_LB_WIN
#define SORT_LB_WIN 16
#endif
// keys per thread / per tile of one onesweep pass (u32: 30-bit keys, u64: 63-bit keys)
template <typename K> struct SortCfg {
    static constexpr int ITEMS = sizeof(K) == 4 ? SORT_ITEMS32 : SORT_ITEMS64;
    static constexpr int TILE = 256 * ITEMS;
};
constexpr int SORT_TILE_MIN = 256 * (SORT_ITEMS32 < SORT_ITEMS64 ? SORT_ITEMS32 : SORT_ITEMS64);
constexpr int RADIX = 256;
constexpr unsigned FLAG_AGG = 1u << 30;
constexpr unsigned FLAG_INC = 2u << 30;
constexpr unsigned VALUE_MASK = (1u << 30) - 1u;

__device__ __forceinline__ void tri_box(const float* t, float lo[3], float hi[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = sel_min(sel_min(t[a], t[3 + a]), t[6 + a]);
        hi[a] = sel_max(sel_max(t[a], t[3 + a]), t[6 + a]);
    }
}

__device__ __forceinline__ void load_tri(const float* tris, int64_t i, float t[9]) {
    const float* p = tris + 9 * i;
#pragma unroll
    for (int k = 0; k < 9; ++k) t[k] = __ldg(p + k);
}

// Gather of one 36-B row by two 256-bit loads of the 32-B aligned 64-B window that
// contains it (the row never straddles more than two sectors: 36 i mod 32 <= 28), then a
// 3-stage barrel shift by the row's offset in the window (i mod 8 floats).  Nine scalar
// loads of the same row issued back to back each go to L2 while the first miss is in
// flight (ncu, 10M emit: 9.5 L2 read sectors per leaf); this asks for exactly two.
// (The scene's row array carries 64 B of slack for the last rows' windows.)
#ifndef RT_WIDE_GATHER
#define RT_WIDE_GATHER 1
#endif
// The gathered row is used once: not allocating it in L1 (L1::no_allocate, or .cg) took the
// 10M emit 0.975 -> 0.946 ms (same box, 2 x 30 builds); L1::evict_first did not help.
#ifndef RT_GATHER_LD
#define RT_GATHER_LD "ld.global.nc.L1::no_allocate.v8.f32"
#endif
__device__ __forceinline__ void ldg256(const float* p, float w[8]) {
    asm(RT_GATHER_LD " {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(w[0]), "=f"(w[1]), "=f"(w[2]), "=f"(w[3]), "=f"(w[4]), "=f"(w[5]), "=f"(w[6]), "=f"(w[7])
        : "l"(p));
}
__device__ __forceinline__ void load_tri_gather(const float* tris, int64_t i, float t[9]) {
#if RT_WIDE_GATHER
    const int64_t e = 9 * i;
    const int o = (int)(e & 7);                 // == i & 7
    float w[16];
    ldg256(tris + (e - o), w);
    ldg256(tris + (e - o) + 8, w + 8);
    float a[12], b[10];
#pragma unroll
    for (int j = 0; j < 12; ++j) a[j] = (o & 4) ? w[j + 4] : w[j];
#pragma unroll
    for (int j = 0; j < 10; ++j) b[j] = (o & 2) ? a[j + 2] : a[j];
#pragma unroll
    for (int j = 0; j < 9; ++j) t[j] = (o & 1) ? b[j + 1] : b[j];
#else
    load_tri(tris, i, t);
#endif
}

// Block-cooperative staging of TRI_CHUNK consecutive triangles (36 B each) into
// shared memory with 16-B coalesced loads; the per-triangle loads of a direct
// (n, 9) walk are 36-B strided and waste most of each sector request.
constexpr int TRI_CHUNK = 256;
__device__ __forceinline__ int stage_tris(const float* __restrict__ tris, int64_t base, int64_t n, float* s) {
    const int64_t left = n - base;
    const int cnt = left < TRI_CHUNK ? (int)left : TRI_CHUNK;
    const int nf = 9 * cnt, nv = nf >> 2;
    const float4* src = reinterpret_cast<const float4*>(tris + 9 * base);   // 9216-B aligned chunks
    for (int k = threadIdx.x; k < nv; k += blockDim.x) reinterpret_cast<float4*>(s)[k] = __ldg(src + k);
    for (int k = 4 * nv + threadIdx.x; k < nf; k += blockDim.x) s[k] = __ldg(tris + 9 * base + k);
    return cnt;
}

// Full chunks are streamed by the TMA bulk engine instead: one thread issues a 9216-B
// cp.async.bulk per chunk into a ring of TRI_STAGES shared buffers, completion is
// signalled on an mbarrier, so TRI_STAGES chunks per block are in flight while the
// block works on the oldest one (the register/LSU path above kept ~2 loads per thread
// in flight and reached ~3.7 TB/s).  The partial tail chunk goes through stage_tris.
#ifndef TRI_STAGES
#define TRI_STAGES 3
#endif
#ifndef TRI_BLOCKS_PER_SM
#define TRI_BLOCKS_PER_SM 4   // 3 stages x 4 blocks: 1M bounds+morton 43.5 -> 34.5 us, 10M 190 -> 151 us
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tma_chunk(float* dst, const float* src, unsigned bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// The chunk loop shared by K1 and K2: body(buf, cnt, base) for each of this block's
// chunks, buf = the chunk's 9 * cnt floats in shared memory.
template <class Body>
__device__ __forceinline__ void for_each_tri_chunk(const float* __restrict__ tris, int64_t n,
                                                   float (*s_tri)[9 * TRI_CHUNK], uint64_t* s_bar, Body&& body) {
    constexpr unsigned CHUNK_BYTES = 9 * TRI_CHUNK * sizeof(float);
    const int64_t nfull = n / TRI_CHUNK, nchunks = (n + TRI_CHUNK - 1) / TRI_CHUNK;
    if (threadIdx.x == 0) {
        for (int k = 0; k < TRI_STAGES; ++k) mbar_init(s_bar + k);
        mbar_init_fence();
        for (int k = 0; k < TRI_STAGES; ++k) {
            const int64_t c = blockIdx.x + (int64_t)k * gridDim.x;
            if (c < nfull) tma_chunk(s_tri[k], tris + 9 * c * TRI_CHUNK, CHUNK_BYTES, s_bar + k);
        }
    }
    __syncthreads();
    int k = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
        const int sidx = k % TRI_STAGES;
        float* buf = s_tri[sidx];
        int cnt = TRI_CHUNK;
        if (c < nfull) {
            mbar_wait(s_bar + sidx, (unsigned)(k / TRI_STAGES) & 1u);
        } else {
            cnt = stage_tris(tris, c * TRI_CHUNK, n, buf);
            __syncthreads();
        }
        body(buf, cnt, c * TRI_CHUNK);
        __syncthreads();                           // the stage is free again
        if (threadIdx.x == 0) {
            const int64_t cn = c + (int64_t)TRI_STAGES * gridDim.x;
            if (cn < nfull) tma_chunk(buf, tris + 9 * cn * TRI_CHUNK, CHUNK_BYTES, s_bar + sidx);
        }
    }
}

// ---- K1 -------------------------------------------------------------------
__global__ void __launch_bounds__(TRI_CHUNK) lbvh_bounds_kernel(const float* __restrict__ tris, int64_t n,
                                                               unsigned int* __restrict__ cb_enc) {
    __shared__ __align__(128) float s_tri[TRI_STAGES][9 * TRI_CHUNK];
    __shared__ __align__(8) uint64_t s_bar[TRI_STAGES];
    pdl_trigger();
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for_each_tri_chunk(tris, n, s_tri, s_bar, [&](const float* buf, int cnt, int64_t) {
        if ((int)threadIdx.x < cnt) {
            float t[9], blo[3], bhi[3];
#pragma unroll
            for (int k = 0; k < 9; ++k) t[k] = buf[9 * threadIdx.x + k];
            tri_box(t, blo, bhi);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                float c = __fmul_rn(0.5f, __fadd_rn(blo[a], bhi[a]));
                lo[a] = sel_min(lo[a], c);
                hi[a] = sel_max(hi[a], c);
            }
        }
    });
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            lo[a] = sel_min(lo[a], __shfl_xor_sync(RT_FULL, lo[a], off));
            hi[a] = sel_max(hi[a], __shfl_xor_sync(RT_FULL, hi[a], off));
        }
    }
    __shared__ float s[8][6];
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) { s[w][a] = lo[a]; s[w][3 + a] = hi[a]; }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        int a = threadIdx.x;
        float v = s[0][a];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) v = (a < 3) ? sel_min(v, s[k][a]) : sel_max(v, s[k][a]);
        // both accumulators start at 0 (one memset with the sort scratch): the min
        // slots hold max(~ord(v)), since ~ord is order-reversing
        if (a < 3) atomicMax(cb_enc + a, ~f2ord(v));
        else atomicMax(cb_enc + a, f2ord(v));
    }
}

// centroid bounds and inverse extents from the accumulators (each Morton block
// computes them; block 0 also stores them for rt_bvh_download)
__device__ __forceinline__ void bounds_from_enc(const unsigned int* __restrict__ cb_enc, float lo[3], float inv[3],
                                                float* __restrict__ cb) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float l = ord2f(~__ldg(cb_enc + a)), h = ord2f(__ldg(cb_enc + 3 + a));
        const float ext = __fsub_rn(h, l);
        lo[a] = l;
        inv[a] = ext > 0.0f ? __fdiv_rn(1.0f, ext) : 0.0f;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            cb[a] = l;
            cb[3 + a] = h;
            cb[6 + a] = inv[a];
        }
    }
}

// ---- K2 -------------------------------------------------------------------
__device__ __forceinline__ uint32_t expand10(uint32_t v) {
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ uint64_t expand21(uint64_t v) {
    v &= 0x1FFFFFull;
    v = (v | (v << 32)) & 0x001F00000000FFFFull;
    v = (v | (v << 16)) & 0x001F0000FF0000FFull;
    v = (v | (v << 8)) & 0x100F00F00F00F00Full;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

// K2 fused with the onesweep digit histogram of every pass (the keys are in
// registers here, so the histogram costs no extra read of the key array)
template <typename K, int B, int PASSES, int DB>
__global__ void __launch_bounds__(TRI_CHUNK) lbvh_morton_kernel(const float* __restrict__ tris, int64_t n,
                                                               const unsigned int* __restrict__ cb_enc,
                                                               float* __restrict__ cb, K* __restrict__ keys,
                                                               unsigned int* __restrict__ hist) {
    constexpr int NB = 1 << DB;                    // digit bins per pass
    __shared__ unsigned int s_hist[PASSES][NB];
    __shared__ __align__(128) float s_tri[TRI_STAGES][9 * TRI_CHUNK];
    __shared__ __align__(8) uint64_t s_bar[TRI_STAGES];
    for (int i = threadIdx.x; i < PASSES * NB; i += blockDim.x) (&s_hist[0][0])[i] = 0;
    const float scale = (float)(1u << B), qmax = (float)((1u << B) - 1u);
    pdl_wait();                                    // K1's centroid bounds
    pdl_trigger();
    float lo[3], inv[3];
    bounds_from_enc(cb_enc, lo, inv, cb);
    for_each_tri_chunk(tris, n, s_tri, s_bar, [&](const float* buf, int cnt, int64_t base) {
        if ((int)threadIdx.x < cnt) {
            float t[9], blo[3], bhi[3];
#pragma unroll
            for (int k = 0; k < 9; ++k) t[k] = buf[9 * threadIdx.x + k];
            tri_box(t, blo, bhi);
            uint32_t q[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                float c = __fmul_rn(0.5f, __fadd_rn(blo[a], bhi[a]));
                float x = __fmul_rn(__fmul_rn(__fsub_rn(c, lo[a]), inv[a]), scale);
                x = sel_min(sel_max(x, 0.0f), qmax);
                q[a] = (uint32_t)x;
            }
            K k;
            if (B == 10)
                k = (K)((expand10(q[0]) << 2) | (expand10(q[1]) << 1) | expand10(q[2]));
            else
                k = (K)((expand21(q[0]) << 2) | (expand21(q[1]) << 1) | expand21(q[2]));
            keys[base + threadIdx.x] = k;
#pragma unroll
            for (int p = 0; p < PASSES; ++p) atomicAdd(&s_hist[p][(unsigned)(k >> (DB * p)) & (NB - 1u)], 1u);
        }
    });
    for (int i = threadIdx.x; i < PASSES * NB; i += blockDim.x) {
        unsigned v = (&s_hist[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

template <typename K, bool BALLOT>
__device__ __forceinline__ void onesweep_pass(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int64_t n, int shift, const unsigned int* __restrict__ hist,
    unsigned int* status, unsigned int* counter) {
    typedef cub::BlockScan<unsigned int, SORT_THREADS> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned int s_warp[SORT_THREADS / 32][RADIX];
    __shared__ unsigned int s_base[RADIX];
    __shared__ unsigned int s_texcl[RADIX];
    constexpr int SORT_ITEMS = SortCfg<K>::ITEMS, SORT_TILE = SortCfg<K>::TILE;
    __shared__ K s_keys[SORT_TILE];
    __shared__ uint32_t s_vals[SORT_TILE];
    __shared__ unsigned int s_tile;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);     // (counters were zeroed before K1)
    for (int w = 0; w < SORT_THREADS / 32; ++w) s_warp[w][tid] = 0;
    pdl_wait();                                        // the previous pass's keys / values
    pdl_trigger();
    __syncthreads();
    const unsigned tile = s_tile;
    const int64_t seg = (int64_t)tile * SORT_TILE + (int64_t)warp * (32 * SORT_ITEMS);

    K key[SORT_ITEMS];
    uint32_t val[SORT_ITEMS];
    unsigned rank[SORT_ITEMS];
    const unsigned lt_mask = (1u << lane) - 1u;
    // all loads, then all warp matches (independent, so their latencies overlap),
    // then the per-digit warp counters in item order (stable ranks)
    unsigned dig[SORT_ITEMS], peers[SORT_ITEMS];
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        int64_t idx = seg + i * 32 + lane;
        bool ok = idx < n;
        key[i] = ok ? keys_in[idx] : (K)0;
        val[i] = ok ? (vals_in ? vals_in[idx] : (uint32_t)idx) : 0u;
    }
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        const bool ok = seg + i * 32 + lane < n;
        dig[i] = ok ? ((unsigned)(key[i] >> shift) & 0xFFu) : 0x100u;
if (BALLOT) {
            // peers by 9 bit-plane ballots (fixed-latency votes) instead of MATCH.ANY:
            // more instructions, but MATCH.ANY's throughput limits the large sorts
            // (10M: 4 passes 0.462 -> 0.425 ms; 1M: 0.071 -> 0.075 ms, latency-bound)
            unsigned pm = RT_FULL;
#pragma unroll
            for (int b = 0; b < 9; ++b) {
                const bool bit = (dig[i] >> b) & 1u;
                const unsigned bb = __ballot_sync(RT_FULL, bit);
                pm &= bit ? bb : ~bb;
            }
            peers[i] = pm;
        } else {
            peers[i] = __match_any_sync(RT_FULL, dig[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        const bool ok = dig[i] < 0x100u;
        const unsigned below = __popc(peers[i] & lt_mask);
        unsigned base = 0;
        if (ok) base = s_warp[warp][dig[i]];
        __syncwarp();
        if (ok && below == 0) s_warp[warp][dig[i]] = base + __popc(peers[i]);
        __syncwarp();
        rank[i] = base + below;
    }
    __syncthreads();
    // per-digit warp prefixes and the tile count (thread == digit)
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < SORT_THREADS / 32; ++w) {
        unsigned c = s_warp[w][tid];
        s_warp[w][tid] = run;
        run += c;
    }
    const unsigned tile_count = run;
    // publish aggregate, look back, publish inclusive prefix
    unsigned* st = status + (size_t)tile * RADIX + tid;
    unsigned excl = 0;
    if (tile == 0) {
        atomicExch(st, FLAG_INC | tile_count);
    } else {
        atomicExch(st, FLAG_AGG | tile_count);
        // windowed look-back: LB_WIN independent status loads per round instead of
        // one dependent L2 round trip per predecessor tile
        constexpr int LB_WIN = SORT_LB_WIN;
        int j = (int)tile - 1;
        bool done = false;
        while (!done) {
            unsigned w[LB_WIN];
#pragma unroll
            for (int k = 0; k < LB_WIN; ++k)
                w[k] = (j - k >= 0) ? *((volatile unsigned*)(status + (size_t)(j - k) * RADIX + tid)) : (2u << 30);
            // consume from the nearest predecessor down to the first inclusive prefix;
            // stop at a not-yet-published entry and re-poll from there
            int k = 0;
            for (; k < LB_WIN; ++k) {
                const unsigned s = w[k];
                if ((s & ~VALUE_MASK) == 0) break;
                excl += s & VALUE_MASK;
                if (s & FLAG_INC) { done = true; break; }
            }
            if (!done) j -= k;
        }
        atomicExch(st, FLAG_INC | (excl + tile_count));
    }
    // global digit base = exclusive scan of the digit histogram + look-back prefix;
    // the tile is first staged in shared memory in digit order (local position =
    // tile-exclusive digit offset + warp offset + rank), then every digit's run is
    // written out contiguously (coalesced) instead of a per-key scatter
    unsigned bin_excl, tile_excl;
    Scan(scan_tmp).ExclusiveSum(hist[tid], bin_excl);
    __syncthreads();
    Scan(scan_tmp).ExclusiveSum(tile_count, tile_excl);
    s_base[tid] = bin_excl + excl - tile_excl;        // + local position = global position
    s_texcl[tid] = tile_excl;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        int64_t idx = seg + i * 32 + lane;
        if (idx < n) {
            unsigned d = (unsigned)(key[i] >> shift) & 0xFFu;
            unsigned lpos = s_texcl[d] + s_warp[warp][d] + rank[i];
            s_keys[lpos] = key[i];
            s_vals[lpos] = val[i];
        }
    }
    __syncthreads();
    const int64_t left = n - (int64_t)tile * SORT_TILE;
    const int cnt = left < SORT_TILE ? (int)left : SORT_TILE;
    for (int j = tid; j < cnt; j += SORT_THREADS) {
        const K k = s_keys[j];
        const unsigned pos = s_base[(unsigned)(k >> shift) & 0xFFu] + (unsigned)j;
        keys_out[pos] = k;
        vals_out[pos] = s_vals[j];
    }
}

// ---- 30-bit keys in three passes of 10-bit digits ------------------------------
// The same tile algorithm as onesweep_pass (bit-plane ballot ranking, decoupled
// look-back, digit-ordered staging, contiguous runs out) with 1024 bins: one pass fewer
// than four 8-bit passes over 30 bits (the last of which sorted 6 bits).  Each thread
// owns 4 adjacent bins: its warp prefixes move as one 64-bit shared load, its look-back
// status words of a predecessor tile are adjacent, and it publishes them with one 128-bit
// store.  Per-warp digit counters are 16-bit (a warp ranks 32 x ITEMS keys).
constexpr int R10 = 1024;
#ifndef SORT_LB_WIN10
#define SORT_LB_WIN10 2   // 1 / 2 / 4 / 8 / 16: 10M sort 0.405 / 0.396 / 0.411 / 0.469 / 0.705 ms
#endif
// Tile geometry of the 10-bit pass (same box, sort ms at 1M / 10M): 256 threads x 12 keys
// 0.065 / 0.369; 512 x 8 0.059 / 0.371; 512 x 12 0.066 / 0.325; 512 x 13 0.062 / 0.319;
// 512 x 14 0.050 / 0.316; 512 x 15 0.051 / 0.320; 512 x 16 (spills) 0.060 / 0.343.  At 1M,
// 7168-key tiles make 140 tiles: one per SM in a single wave (13 keys: 151 tiles, some SMs
// take two).  Twice the threads per tile halve the tiles a look-back chain crosses.
#ifndef SORT_ITEMS10
#define SORT_ITEMS10 14   // keys per thread
#endif
#ifndef SORT_THREADS10
#define SORT_THREADS10 512  // threads per tile of the 10-bit pass (256: 4 bins per thread; 512: 2)
#endif
constexpr int TILE10 = SORT_THREADS10 * SORT_ITEMS10;
#ifndef SORT_LB_SLEEP
#define SORT_LB_SLEEP 0
#endif
// a thread's PER adjacent look-back status words as one relaxed vector access
template <int PER>
__device__ __forceinline__ void ld_status_n(const unsigned* p, unsigned (&v)[PER]) {
    if constexpr (PER == 4) {
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "l"(p)
                     : "memory");
    } else if constexpr (PER == 2) {
        asm volatile("ld.relaxed.gpu.global.v2.u32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "l"(p) : "memory");
    } else {
        static_assert(PER == 1, "1, 2 or 4 bins per thread");
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v[0]) : "l"(p) : "memory");
    }
}
template <int PER>
__device__ __forceinline__ void st_status_n(unsigned* p, const unsigned (&v)[PER]) {
    if constexpr (PER == 4) {
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                     "r"(v[3])
                     : "memory");
    } else if constexpr (PER == 2) {
        asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v[0]), "r"(v[1]) : "memory");
    } else {
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v[0]) : "memory");
    }
}

#ifndef RT_SORT_TL
#define RT_SORT_TL 0          // diagnostic builds: per-tile phase timestamps of the last wide pass
#endif
#if RT_SORT_TL
#define RT_SORT_TL_TILES 4096
__device__ unsigned long long g_sort_tl[5 * RT_SORT_TL_TILES];
__device__ __forceinline__ unsigned long long sort_tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SORT_TL_MARK(k, v) \
    if (threadIdx.x == 0 && sm.tile < RT_SORT_TL_TILES) g_sort_tl[5 * sm.tile + (k)] = (v)
#else
#define SORT_TL_MARK(k, v)
#endif

// shared-memory layout of the 10-bit pass (dynamic: 86 KB at 512 threads)
// K: key type; T threads per tile; DB digit bits (1 << DB bins); ITEMS keys per thread
template <typename K, int T, int DB, int ITEMS_>
struct SortWSmem {
    typedef cub::BlockScan<unsigned int, T> Scan;
    static constexpr int R = 1 << DB, ITEMS = ITEMS_, TILE = T * ITEMS_;
    typename Scan::TempStorage scan_tmp;
    alignas(16) unsigned short warp[T / 32][R];
    unsigned int base[R];
    unsigned short texcl[R];
    K keys[TILE];
    uint32_t vals[TILE];
    unsigned int tile;
};

template <typename K, int T, int DB, int ITEMS_>
__device__ __forceinline__ void onesweep_wide_pass(const K* __restrict__ keys_in,
                                                   const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
                                                   uint32_t* __restrict__ vals_out, int64_t n, int shift,
                                                   const unsigned int* __restrict__ hist, unsigned int* status,
                                                   unsigned int* counter) {
    typedef SortWSmem<K, T, DB, ITEMS_> SM;
    typedef typename SM::Scan Scan;
    constexpr int ITEMS = SM::ITEMS, TILE = SM::TILE, R10 = SM::R, PER = R10 / T;
    extern __shared__ __align__(16) unsigned char sort10_smem[];
    SM& sm = *reinterpret_cast<SM*>(sort10_smem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#if RT_SORT_TL
    const unsigned long long tl0 = sort_tl_now();
#endif
    if (tid == 0) sm.tile = atomicAdd(counter, 1u);
    {
        uint4* z = reinterpret_cast<uint4*>(&sm.warp[0][0]);
        constexpr int NZ = (int)(sizeof(sm.warp) / sizeof(uint4));
#pragma unroll
        for (int k = tid; k < NZ; k += T) z[k] = make_uint4(0, 0, 0, 0);
    }
    pdl_wait();
    pdl_trigger();
    __syncthreads();
    SORT_TL_MARK(0, tl0);
    SORT_TL_MARK(1, sort_tl_now());
    const unsigned tile = sm.tile;
    const int64_t seg = (int64_t)tile * TILE + (int64_t)warp * (32 * ITEMS);
    K key[ITEMS];
    uint32_t val[ITEMS];
    unsigned dig[ITEMS], peers[ITEMS], rank[ITEMS];
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int64_t idx = seg + i * 32 + lane;
        const bool ok = idx < n;
        key[i] = ok ? keys_in[idx] : (K)0;
        val[i] = ok ? (vals_in ? vals_in[idx] : (uint32_t)idx) : 0u;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        // keys past n take the last bin: they follow every real key in the stable order, so
        // they land behind the tile's real keys and are never written out
        const bool ok = seg + i * 32 + lane < n;
        dig[i] = ok ? ((unsigned)(key[i] >> shift) & (R10 - 1u)) : (R10 - 1u);
        unsigned pm = RT_FULL;
#pragma unroll
        for (int b = 0; b < DB; ++b) {
            const bool bit = (dig[i] >> b) & 1u;
            const unsigned bb = __ballot_sync(RT_FULL, bit);
            pm &= bit ? bb : ~bb;
        }
        peers[i] = pm;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const unsigned below = __popc(peers[i] & lt_mask);
        const unsigned base = sm.warp[warp][dig[i]];
        __syncwarp();
        if (below == 0) sm.warp[warp][dig[i]] = (unsigned short)(base + __popc(peers[i]));
        __syncwarp();
        rank[i] = base + below;
    }
    __syncthreads();
    SORT_TL_MARK(2, sort_tl_now());
    // warp prefixes of this thread's PER bins; tc = the tile's count per bin
    unsigned tc[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) tc[j] = 0;
#pragma unroll
    for (int w = 0; w < T / 32; ++w) {
        if constexpr (PER == 4) {
            uint2* pw = reinterpret_cast<uint2*>(&sm.warp[w][PER * tid]);
            const uint2 v = *pw;
            const unsigned c[4] = {v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16};
            *pw = make_uint2(tc[0] | (tc[1] << 16), tc[2] | (tc[3] << 16));
#pragma unroll
            for (int j = 0; j < 4; ++j) tc[j] += c[j];
        } else if constexpr (PER == 2) {
            unsigned* pw = reinterpret_cast<unsigned*>(&sm.warp[w][PER * tid]);
            const unsigned v = *pw;
            *pw = tc[0] | (tc[1] << 16);
            tc[0] += v & 0xFFFFu;
            tc[1] += v >> 16;
        } else {
            const unsigned v = sm.warp[w][tid];
            sm.warp[w][tid] = (unsigned short)tc[0];
            tc[0] += v;
        }
    }
    // publish aggregates, look back, publish inclusive prefixes.  A predecessor's thread
    // publishes its PER bins in one vector store, so the status words it holds are always of
    // one kind (all unpublished, all aggregate or all inclusive): the thread walks back over
    // predecessors with one vector load each
    unsigned* st = status + (size_t)tile * R10 + PER * tid;
    unsigned excl[PER], pub[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) excl[j] = 0;
    if (tile == 0) {
#pragma unroll
        for (int j = 0; j < PER; ++j) pub[j] = FLAG_INC | tc[j];
        st_status_n<PER>(st, pub);
    } else {
#pragma unroll
        for (int j = 0; j < PER; ++j) pub[j] = FLAG_AGG | tc[j];
        st_status_n<PER>(st, pub);
        constexpr int LB = SORT_LB_WIN10;
        int j = (int)tile - 1;
        bool done = false;
        while (!done) {
            unsigned w[LB][PER];
#pragma unroll
            for (int k = 0; k < LB; ++k) {
                if (j - k >= 0) {
                    ld_status_n<PER>(status + (size_t)(j - k) * R10 + PER * tid, w[k]);
                } else {
#pragma unroll
                    for (int q = 0; q < PER; ++q) w[k][q] = 0;
                }
            }
            int k = 0;
#pragma unroll
            for (int kk = 0; kk < LB; ++kk) {
                if (done || k < kk) continue;            // stopped earlier in this window
                const unsigned f = w[kk][0] & ~VALUE_MASK;
                unsigned mixed = 0;                      // (defensively: a vector store seen half-way)
#pragma unroll
                for (int q = 1; q < PER; ++q) mixed |= (w[kk][0] ^ w[kk][q]);
                if (f == 0 || (mixed & ~VALUE_MASK)) continue;   // not yet published: re-poll
#pragma unroll
                for (int q = 0; q < PER; ++q) excl[q] += w[kk][q] & VALUE_MASK;
                k = kk + 1;
                if (f & FLAG_INC) done = true;
            }
            j -= k;
#if SORT_LB_SLEEP
            if (k == 0) __nanosleep(SORT_LB_SLEEP);   // no progress: back off instead of hammering L2
#endif
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) pub[q] = FLAG_INC | (excl[q] + tc[q]);
        st_status_n<PER>(st, pub);
    }
    unsigned hv[PER], bin_excl[PER], tile_excl[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) hv[q] = __ldg(hist + PER * tid + q);
    Scan(sm.scan_tmp).ExclusiveSum(hv, bin_excl);
    __syncthreads();
    SORT_TL_MARK(3, sort_tl_now());
    Scan(sm.scan_tmp).ExclusiveSum(tc, tile_excl);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        sm.base[PER * tid + q] = bin_excl[q] + excl[q] - tile_excl[q];
        sm.texcl[PER * tid + q] = (unsigned short)tile_excl[q];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const unsigned lpos = sm.texcl[dig[i]] + sm.warp[warp][dig[i]] + rank[i];
        sm.keys[lpos] = key[i];
        sm.vals[lpos] = val[i];
    }
    __syncthreads();
    const int64_t left = n - (int64_t)tile * TILE;
    const int cnt = left < TILE ? (int)left : TILE;
    for (int j = tid; j < cnt; j += T) {
        const K k = sm.keys[j];
        const unsigned pos = sm.base[(unsigned)(k >> shift) & (R10 - 1u)] + (unsigned)j;
        keys_out[pos] = k;
        vals_out[pos] = sm.vals[j];
    }
#if RT_SORT_TL
    __syncthreads();
    SORT_TL_MARK(4, sort_tl_now());
#endif
}
// 30-bit keys: 3 passes of 10-bit digits
typedef SortWSmem<uint32_t, SORT_THREADS10, 10, SORT_ITEMS10> Sort10Smem;
__global__ void __launch_bounds__(SORT_THREADS10, 1024 / SORT_THREADS10) onesweep10_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int64_t n, int shift, const unsigned int* __restrict__ hist, unsigned int* status,
    unsigned int* counter) {
    onesweep_wide_pass<uint32_t, SORT_THREADS10, 10, SORT_ITEMS10>(keys_in, vals_in, keys_out, vals_out, n, shift,
                                                                    hist, status, counter);
}
// 63-bit keys: 7 passes of 9-bit digits (RT_SORT9), 512 threads per tile.  Keys per thread by
// size (same box, sort ms at 1M / 10M): 6: 0.146 / 0.891; 8: 0.129 / 0.809; 10: 0.142 / 0.775;
// 12: 0.155 / 0.763 (8 x 8-bit passes: 0.137 / 0.904) -- 8 below SORT9_BIG_N keys, 12 above
#ifndef SORT_THREADS9
#define SORT_THREADS9 512
#endif
#ifndef SORT_ITEMS9
#define SORT_ITEMS9 8
#endif
#ifndef SORT_ITEMS9_BIG
#define SORT_ITEMS9_BIG 12
#endif
#ifndef SORT9_BIG_N
#define SORT9_BIG_N (1 << 22)
#endif
constexpr int TILE9 = SORT_THREADS9 * SORT_ITEMS9;
constexpr int TILE9_BIG = SORT_THREADS9 * SORT_ITEMS9_BIG;
template <int ITEMS>
__global__ void __launch_bounds__(SORT_THREADS9, 1024 / SORT_THREADS9) onesweep9_kernel(
    const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint64_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int64_t n, int shift, const unsigned int* __restrict__ hist, unsigned int* status,
    unsigned int* counter) {
    onesweep_wide_pass<uint64_t, SORT_THREADS9, 9, ITEMS>(keys_in, vals_in, keys_out, vals_out, n, shift, hist,
                                                           status, counter);
}

// 30-bit keys: 64 registers -> 4 blocks per SM (10M: 4 passes 0.427 -> 0.391 ms); 63-bit
// keys keep the single-argument bound (an explicit minBlocks = 1 costs 15 % there).
#define ONESWEEP_ARGS                                                                                  \
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,   \
        uint32_t* __restrict__ vals_out, int64_t n, int shift, const unsigned int* __restrict__ hist, \
        unsigned int *status, unsigned int *counter
template <bool BALLOT, typename K = uint32_t>
__global__ void __launch_bounds__(SORT_THREADS, 4) onesweep32_kernel(ONESWEEP_ARGS) {
    onesweep_pass<K, BALLOT>(keys_in, vals_in, keys_out, vals_out, n, shift, hist, status, counter);
}
template <bool BALLOT, typename K = uint64_t>
__global__ void __launch_bounds__(SORT_THREADS) onesweep64_kernel(ONESWEEP_ARGS) {
    onesweep_pass<K, BALLOT>(keys_in, vals_in, keys_out, vals_out, n, shift, hist, status, counter);
}
#undef ONESWEEP_ARGS

// ---- K4+K5: fused Karras emission + bottom-up refit ------------------------
// One thread per leaf climbs the tree (Apetrei 2014's agglomerative scheme):
// a node covering keys [l, r] is the LEFT child of its parent iff
// delta(r, r+1) > delta(l-1, l) (the parent's split is the boundary with the
// longer common prefix; no ties exist for index-augmented keys).  Siblings meet
// at the parent's split slot gamma with one acq_rel exchange of their far
// endpoints: the first arrival publishes its box and leaves, the second builds
// the parent.  Karras's node numbering (internal 0..n-2, root 0) is recovered
// exactly: a left child is numbered by its right end, a right child by its
// left end, so child/parent arrays equal the split-search construction bit for
// bit (oracle/rt_oracle.c orc_lbvh_karras + orc_lbvh_refit).
//
// node layout (Aila-Laine): n0 = (L.lo.x, L.hi.x, L.lo.y, L.hi.y)
//                           n1 = (R.lo.x, R.hi.x, R.lo.y, R.hi.y)
//                           n2 = (L.lo.z, L.hi.z, R.lo.z, R.hi.z)
//                           n3 = (left id, right id, height, 0)   id < 0: ~leaf
template <typename K>
__device__ __forceinline__ int adj_delta(const K* __restrict__ k, int64_t n, int64_t i) {
    // delta(i, i+1); -1 outside [0, n-2]
    if (i < 0 || i >= n - 1) return -1;
    K a = k[i], b = k[i + 1];
    if (a != b) return (sizeof(K) == 8) ? __clzll((unsigned long long)(a ^ b)) : __clz((unsigned)(a ^ b));
    return (int)(8 * sizeof(K)) + __clz((unsigned)i ^ (unsigned)(i + 1));
}

#include "emit.cuh"

// n == 1: a root whose left child is leaf 0 and whose right box is empty
__global__ void single_leaf_root(const float* tris, const uint32_t* mask, float4* nodes, float4* tri_sorted,
                                 float4* leaf_box, uint32_t* order) {
    float t[9], lo[3], hi[3];
    load_tri(tris, 0, t);
    tri_box(t, lo, hi);
    order[0] = 0;
    tri_sorted[0] = make_float4(t[0], t[1], t[2], __int_as_float(0));
    tri_sorted[1] = make_float4(t[3], t[4], t[5], __uint_as_float(mask[0]));
    tri_sorted[2] = make_float4(t[6], t[7], t[8], 0.0f);
    leaf_box[0] = make_float4(lo[0], lo[1], lo[2], 0.f);
    leaf_box[1] = make_float4(hi[0], hi[1], hi[2], 0.f);
    nodes[0] = make_float4(lo[0], hi[0], lo[1], hi[1]);
    nodes[1] = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);    // empty: never hit
    nodes[2] = make_float4(lo[2], hi[2], INFINITY, INFINITY);
    nodes[3] = make_float4(__int_as_float(~0), __int_as_float(~0), __int_as_float(1), 0.0f);
}

// DB: digit bits per onesweep pass (30-bit keys: 3 x 10 with RT_SORT10, else 4 x 8;
// 63-bit keys: 8 x 8)
#ifndef RT_SORT10
#define RT_SORT10 1
#endif
#ifndef RT_SORT9
#define RT_SORT9 1          // 63-bit keys: 7 passes of 9-bit digits (else 8 x 8 bits)
#endif
template <typename K, int PASSES, int B, int DB>
int build_typed(rt_ctx* ctx, rt_scene* s) {
    const int64_t n = s->n;
    cudaStream_t st = ctx->stream;
    const int grid_stream = ctx->num_sms * TRI_BLOCKS_PER_SM;
    constexpr int NB = 1 << DB;
    // the sort scratch (digit histograms, tile counters, the centroid-bound accumulators and
    // the look-back status) arrives zeroed: at allocation, then by the previous build's
    // lbvh_emit_global_kernel
    int gb = (int)((n + 255) / 256);
    if (gb > grid_stream) gb = grid_stream;
    const bool big9 = DB == 9 && n >= SORT9_BIG_N;
    const int64_t TILE = DB == 10 ? TILE10 : (DB == 9 ? (big9 ? TILE9_BIG : TILE9) : SortCfg<K>::TILE);
    const int64_t tiles = (n + TILE - 1) / TILE;
    unsigned int* hist = s->sort_scratch;                    // PASSES * NB
    unsigned int* counters = hist + PASSES * NB;             // [0, 8) tile counters, [8, 14) cb_enc, [16] emit count
    unsigned int* cb_enc = counters + 8;
    unsigned int* status = counters + 32;                    // PASSES * tiles * NB
    RT_PROF(ctx, 0);
    // K1
    lbvh_bounds_kernel<<<gb, 256, 0, st>>>(s->tris, n, cb_enc);
    // K2
    K* ka = (K*)s->keys_a;
    K* kb = (K*)s->keys_b;
    RT_PROF(ctx, 1);
    RT_CUDA_TRY(launch_pdl(lbvh_morton_kernel<K, B, PASSES, DB>, gb, 256, st, s->tris, n, cb_enc, s->cbounds, ka, hist));
    RT_PROF(ctx, 2);
    // K3 (digit histograms already accumulated by K2)
    K* kin = ka; K* kout = kb;
    uint32_t* vin = nullptr; uint32_t* vout = s->vals_b;
    RT_PROF(ctx, 3);
#ifndef SORT_BALLOT_MIN
#define SORT_BALLOT_MIN (1 << 21)
#endif
    const bool ballot = sizeof(K) == 8 || n >= SORT_BALLOT_MIN;
    for (int p = 0; p < PASSES; ++p) {
        auto launch = [&](auto kern) {
            return launch_pdl(kern, (unsigned)tiles, SORT_THREADS, st, kin, vin, kout, vout, n, DB * p,
                              hist + p * NB, status + (size_t)p * tiles * NB, counters + p);
        };
        if constexpr (DB == 10 || DB == 9) {
            auto go = [&](auto kern, size_t smem, int threads, bool* attr_set) -> int {
                if (!attr_set[ctx->device & 63]) {     // the opt-in is per device
                    RT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    attr_set[ctx->device & 63] = true;
                }
                RT_CUDA_TRY(launch_pdl_smem(kern, (unsigned)tiles, threads, smem, st, kin, vin, kout, vout, n, DB * p,
                                            hist + p * NB, status + (size_t)p * tiles * NB, counters + p));
                return RT_OK;
            };
            static bool set10[64] = {}, set9[64] = {}, set9b[64] = {};
            int rc;
            if constexpr (DB == 10) {
                rc = go(onesweep10_kernel, sizeof(Sort10Smem), SORT_THREADS10, set10);
            } else if (big9) {
                rc = go(onesweep9_kernel<SORT_ITEMS9_BIG>, sizeof(SortWSmem<uint64_t, SORT_THREADS9, 9, SORT_ITEMS9_BIG>),
                        SORT_THREADS9, set9b);
            } else {
                rc = go(onesweep9_kernel<SORT_ITEMS9>, sizeof(SortWSmem<uint64_t, SORT_THREADS9, 9, SORT_ITEMS9>),
                        SORT_THREADS9, set9);
            }
            if (rc) return rc;
        } else if constexpr (sizeof(K) == 4) {
            RT_CUDA_TRY(ballot ? launch(onesweep32_kernel<true>) : launch(onesweep32_kernel<false>));
        } else {
            RT_CUDA_TRY(launch(onesweep64_kernel<true>));
        }
        K* tk = kin; kin = kout; kout = tk;
        uint32_t* nv = (vout == s->vals_b) ? s->vals_a : s->vals_b;
        vin = vout; vout = nv;
    }
    if (PASSES & 1) {
        // an odd pass count leaves the sorted keys / order in the b buffers: the scene's
        // a / b buffers trade places so keys_a / vals_a hold them (download, scene copy)
        std::swap(s->keys_a, s->keys_b);
        std::swap(s->vals_a, s->vals_b);
    }
    // sorted keys in keys_a (== kin), values in vals_a (== vin)
    // K4 + K5
    RT_PROF(ctx, 4);
    // (the global split slots are reset by the emit kernel at its hand-off boundaries)
    RT_PROF(ctx, 5);
    EmitNode* items = (EmitNode*)s->emit_items;
    const int64_t n_blocks = (n + EMIT_T - 1) / EMIT_T;
    RT_CUDA_TRY(launch_pdl(lbvh_emit_kernel<K>, (unsigned)n_blocks, EMIT_T, st, (const K*)kin, (const uint32_t*)vin,
                           (const float*)s->tris, s->mask_uniform ? (const uint32_t*)nullptr : (const uint32_t*)s->tri_mask,
                           s->mask_value, n, s->child, s->tri_sorted, s->nodes,
                           s->bvh4, items, s->seg_count, (int*)s->flags, s->leaf_box));
    RT_CUDA_TRY(launch_pdl(lbvh_emit_global_kernel<K>, (unsigned)((n_blocks * 32 + 127) / 128), 128u, st,
                           (const K*)kin, n, s->child, s->nodes, s->bvh4, (int*)s->flags, s->leaf_box,
                           (const EmitNode*)items, (const unsigned int*)s->seg_count, n_blocks,
                           reinterpret_cast<uint4*>(s->sort_scratch), (int64_t)(s->sort_scratch_words / 4)));
    RT_PROF(ctx, 6);
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

}  // namespace

int rt_lbvh_build_impl(rt_ctx* ctx, rt_scene* s, int bits) {
    if (s->n == 1) {
        single_leaf_root<<<1, 1, 0, ctx->stream>>>(s->tris, s->tri_mask, s->nodes, s->tri_sorted, s->leaf_box,
                                                   s->vals_a);
        bvh4_single_leaf_kernel<<<1, 1, 0, ctx->stream>>>(s->nodes, s->bvh4);
        RT_CUDA_TRY(cudaGetLastError());
        return RT_OK;
    }
#if RT_SORT10
    if (bits == 30) return build_typed<uint32_t, 3, 10, 10>(ctx, s);
#else
    if (bits == 30) return build_typed<uint32_t, 4, 10, 8>(ctx, s);
#endif
#if RT_SORT9
    return build_typed<uint64_t, 7, 21, 9>(ctx, s);
#else
    return build_typed<uint64_t, 8, 21, 8>(ctx, s);
#endif
}

size_t rt_sort_scratch_words(int64_t n) {
    const int64_t tiles = (n + SORT_TILE_MIN - 1) / SORT_TILE_MIN;
    const int64_t tiles32 = (n + TILE10 - 1) / TILE10;
    const size_t w8 = (size_t)8 * RADIX + 32 + (size_t)8 * tiles * RADIX;
    const size_t w10 = (size_t)3 * R10 + 32 + (size_t)3 * tiles32 * R10;
    const int64_t tiles64 = (n + TILE9 - 1) / TILE9;
    const size_t w9 = (size_t)7 * 512 + 32 + (size_t)7 * tiles64 * 512;
    size_t w = w8 > w10 ? w8 : w10;
    if (w9 > w) w = w9;
    return (w + 3) & ~(size_t)3;        // whole 16-B units (zeroed as uint4 by the emit hand-off)
}

#if RT_SORT_TL
extern "C" int rt_debug_sort_timeline(unsigned long long* out, int32_t n_tiles) {
    if (n_tiles > RT_SORT_TL_TILES) n_tiles = RT_SORT_TL_TILES;
    RT_CUDA_TRY(cudaMemcpyFromSymbol(out, g_sort_tl, sizeof(unsigned long long) * 5 * n_tiles));
    return RT_OK;
}
#endif
