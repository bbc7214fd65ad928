// tlas.cu -- two-level (TLAS / BLAS) closest- and any-hit traversal on the GPU
// (replaces the reference's Tlas / Blas / Instance kernels, accel.py:211-283,
// 439-549, 575-699, 762-895).
//
// A BLAS is an rt_scene in LOCAL space (its own LBVH; triangle prims, or the
// AABBs of custom primitives).  The TLAS is an rt_scene whose primitives are
// the instances' world AABBs (the corners of the BLAS root box through the
// instance matrix, accel.py:459-469), so it reuses the same LBVH builder.
// One thread per ray walks the TLAS 4-wide; at an instance leaf (mask AND,
// accel.py:796) the ray goes to local space (accel.py:804-809; the direction
// keeps its length so local t == world t) and walks that BLAS with a second
// stack.  The tie rule is the reference's: lowest instance, then lowest prim
// (accel.py:629, 815-817).  Normals leave the kernel as (inst, prim) and are
// produced in float64 by the expand kernel: the BLAS's float64 local normal
// (or the sphere's at the hit) through the instance inverse transpose,
// renormalised (accel.py:843-847).  Custom primitives are spheres behind the
// registry: with no registered data, reaching one is RT_EUNSUPPORTED.
#include <map>
#include <vector>

#include "hostio.cuh"
#include "traverse.cuh"

struct BlasDev {
    const float4* bvh4;
    const float4* tris;       // leaf-ordered: v0.w = prim, v1.w = mask (full)
    const double* lnormal;    // (n, 3) float64 local normals (triangles)
    const double* lrows;      // (n, 9) float64 local vertices (nullable): exact (t, u, v) refinement
    const double* data;       // custom: rows (cx, cy, cz, r) of this BLAS's prims (nullptr: not registered)
    int root4, height, kind, geom_type;
};

struct InstDev {
    float inv[12];            // fp32 inverse for the local ray of the walk
    double inv64[12];         // float64 inverse (custom tests, normals)
    uint32_t mask;
    int blas;
    int pad0, pad1;
};

struct rt_tlas {
    int n_inst = 0;
    rt_scene* top = nullptr;            // owned: LBVH over instance world boxes
    std::vector<rt_scene*> blas;        // unique BLAS handles (not owned)
    std::vector<int> inst_blas;
    std::vector<BlasDev> hblas;
    std::vector<InstDev> hinst;
    BlasDev* d_blas = nullptr;
    InstDev* d_inst = nullptr;
    std::vector<double*> d_data;        // per BLAS registered custom rows (owned)
    int top_root4 = 0, top_height = 0, max_height = 0;
};

namespace {

constexpr int TL_THREADS = 128;

struct TlasView {
    const float4* tbvh4;
    const float4* ttris;
    int troot;
    const InstDev* inst;
    const BlasDev* blas;
    int* err;
};

struct Hit2 {
    float t;
    int inst, prim;
    float u, v;
};

// tie bound for the BLAS walk of instance i given the best hit so far: a hit at
// exactly best_t wins iff i < best_inst (each instance is one TLAS leaf, so
// i != best_inst); tri_test rejects a tie when prim >= bound
__device__ __forceinline__ int tie_bound(int i, int best_inst) {
    return (best_inst >= 0 && i < best_inst) ? INT_MAX : INT_MIN;
}

__device__ __forceinline__ void inst_local(const InstDev* __restrict__ I, const RayPre& W, float lo[3], float ld[3]) {
    float m[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) m[k] = __ldg(I->inv + k);
    lo[0] = fmaf(m[0], W.ox, fmaf(m[1], W.oy, fmaf(m[2], W.oz, m[3])));
    lo[1] = fmaf(m[4], W.ox, fmaf(m[5], W.oy, fmaf(m[6], W.oz, m[7])));
    lo[2] = fmaf(m[8], W.ox, fmaf(m[9], W.oy, fmaf(m[10], W.oz, m[11])));
    ld[0] = fmaf(m[0], W.dx, fmaf(m[1], W.dy, m[2] * W.dz));
    ld[1] = fmaf(m[4], W.dx, fmaf(m[5], W.dy, m[6] * W.dz));
    ld[2] = fmaf(m[8], W.dx, fmaf(m[9], W.dy, m[10] * W.dz));
}

// custom primitive (sphere) k of a custom BLAS: float64 test on the float64 local ray
static __device__ __noinline__ double custom_hit(const InstDev* __restrict__ I, const double* __restrict__ row,
                                                 const RayPre& W, double t_min, double t_max) {
    double m[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) m[k] = __ldg(I->inv64 + k);
    double o[3], d[3];
    to_local_f64(m, W.ox, W.oy, W.oz, W.dx, W.dy, W.dz, o, d);
    return sphere_solve_f64(o, d, __ldg(row), __ldg(row + 1), __ldg(row + 2), __ldg(row + 3), t_min, t_max);
}

template <bool STATS>
__device__ __forceinline__ Hit2 tlas_closest(const TlasView& T, const RayPre& W, float tmax, uint32_t ray_mask,
                                             int2* st_top, int2* st_bot, uint32_t& n_tests, uint32_t& n_visits) {
    Hit2 best;
    best.t = tmax; best.inst = -1; best.prim = -1; best.u = 0.f; best.v = 0.f;
    walk4<STATS>(T.tbvh4, T.troot, W, best.t, st_top, n_visits, [&](int k) {
        const float4* tp = T.ttris + 3 * k;
        const int i = __float_as_int(__ldg(tp).w);
        const uint32_t m = __float_as_uint(__ldg(tp + 1).w);
        if (!(m & ray_mask)) return;                          // accel.py:796
        const InstDev* I = T.inst + i;
        const BlasDev B = T.blas[__ldg(&I->blas)];
        float t = best.t, u = best.u, v = best.v;
        int id = tie_bound(i, best.inst);
        const int id0 = id;
        float lo[3], ld[3];
        inst_local(I, W, lo, ld);
        RayPre L;
        ray_setup(L, lo[0], lo[1], lo[2], ld[0], ld[1], ld[2], W.tmin);
        if (B.kind == 0) {
            walk4<STATS>(B.bvh4, B.root4, L, t, st_bot, n_visits, [&](int kk) {
                const float4* q = B.tris + 3 * kk;
                const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
                if (STATS) ++n_tests;
                tri_test(L, a, b, c, t, id, u, v);
            });
        } else {
            if (!B.data) {                                    // accel.py:800-803
                atomicExch(T.err, RT_EUNSUPPORTED);
                return;
            }
            walk4<STATS>(B.bvh4, B.root4, L, t, st_bot, n_visits, [&](int kk) {
                const int prim = __float_as_int(__ldg(B.tris + 3 * kk).w);
                if (STATS) ++n_tests;
                const double th = custom_hit(I, B.data + 4 * (int64_t)prim, W, (double)W.tmin, (double)t);
                if (th < 0.0) return;
                const float tf = (float)th;
                if (tf > t || (tf == t && prim >= id)) return;
                t = tf; id = prim; u = 0.f; v = 0.f;
            });
        }
        if (id != id0) {
            best.t = t; best.inst = i; best.prim = id; best.u = u; best.v = v;
        }
    });
    if (best.inst < 0) best.t = -1.0f;
    return best;
}

__device__ __forceinline__ bool tlas_any(const TlasView& T, const RayPre& W, float tmax, uint32_t ray_mask,
                                         int* st_top, int* st_bot) {
    return walk_any4(T.tbvh4, T.troot, W, tmax, st_top, [&](int k) -> bool {
        const float4* tp = T.ttris + 3 * k;
        const int i = __float_as_int(__ldg(tp).w);
        const uint32_t m = __float_as_uint(__ldg(tp + 1).w);
        if (!(m & ray_mask)) return false;
        const InstDev* I = T.inst + i;
        const BlasDev B = T.blas[__ldg(&I->blas)];
        float lo[3], ld[3];
        inst_local(I, W, lo, ld);
        RayPre L;
        ray_setup(L, lo[0], lo[1], lo[2], ld[0], ld[1], ld[2], W.tmin);
        if (B.kind == 0)
            return walk_any4(B.bvh4, B.root4, L, tmax, st_bot, [&](int kk) -> bool {
                const float4* q = B.tris + 3 * kk;
                return tri_any(L, __ldg(q), __ldg(q + 1), __ldg(q + 2), tmax);
            });
        if (!B.data) {
            atomicExch(T.err, RT_EUNSUPPORTED);
            return false;
        }
        return walk_any4(B.bvh4, B.root4, L, tmax, st_bot, [&](int kk) -> bool {
            const int prim = __float_as_int(__ldg(B.tris + 3 * kk).w);
            return custom_hit(I, B.data + 4 * (int64_t)prim, W, (double)W.tmin, (double)tmax) >= 0.0;
        });
    });
}

template <bool STATS>
__global__ void __launch_bounds__(TL_THREADS) tlas_closest_kernel(const TlasView T, int max_height, int64_t n,
                                                                  const float* __restrict__ rays,
                                                                  float4* __restrict__ hits, uint32_t ray_mask,
                                                                  uint32_t* __restrict__ stats, unsigned int* counter) {
    if (max_height + 1 > RT_STACK) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(T.err, RT_EDEPTH);
        return;
    }
    int2 st_top[RT_STACK4], st_bot[RT_STACK4];
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(counter, 32u);
        base = __shfl_sync(RT_FULL, base, 0);
        if ((int64_t)base >= n) break;
        const int64_t i = (int64_t)base + lane;
        if (i < n) {
            const TraceRay r = load_ray(rays, i);
            RayPre W;
            ray_setup(W, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, r.tmin);
            uint32_t nt = 0, nv = 0;
            const Hit2 h = tlas_closest<STATS>(T, W, r.tmax, ray_mask, st_top, st_bot, nt, nv);
            hits[2 * i] = make_float4(h.t, __int_as_float(h.inst), __int_as_float(h.prim), h.u);
            hits[2 * i + 1] = make_float4(h.v, 0.f, 0.f, 0.f);
            if (STATS) reinterpret_cast<uint2*>(stats)[i] = make_uint2(nt, nv);
        }
    }
}

__global__ void __launch_bounds__(TL_THREADS) tlas_any_kernel(const TlasView T, int max_height, int64_t n,
                                                              const float* __restrict__ rays, uint8_t* __restrict__ out,
                                                              uint32_t ray_mask, unsigned int* counter) {
    if (max_height + 1 > RT_STACK) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(T.err, RT_EDEPTH);
        return;
    }
    int st_top[RT_STACK4], st_bot[RT_STACK4];
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(counter, 32u);
        base = __shfl_sync(RT_FULL, base, 0);
        if ((int64_t)base >= n) break;
        const int64_t i = (int64_t)base + lane;
        if (i < n) {
            const TraceRay r = load_ray(rays, i);
            RayPre W;
            ray_setup(W, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, r.tmin);
            out[i] = tlas_any(T, W, r.tmax, ray_mask, st_top, st_bot) ? 1 : 0;
        }
    }
}

// accel.py:843-847 in the reference's operation order (float64, no contraction)
__device__ __forceinline__ void world_normal_f64(const double* m, double lx, double ly, double lz, double* out) {
    const double wx = __dadd_rn(__dadd_rn(__dmul_rn(m[0], lx), __dmul_rn(m[4], ly)), __dmul_rn(m[8], lz));
    const double wy = __dadd_rn(__dadd_rn(__dmul_rn(m[1], lx), __dmul_rn(m[5], ly)), __dmul_rn(m[9], lz));
    const double wz = __dadd_rn(__dadd_rn(__dmul_rn(m[2], lx), __dmul_rn(m[6], ly)), __dmul_rn(m[10], lz));
    const double il = __ddiv_rn(1.0, sqrt(__dadd_rn(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)),
                                                   __dmul_rn(wz, wz))));
    out[0] = __dmul_rn(wx, il); out[1] = __dmul_rn(wy, il); out[2] = __dmul_rn(wz, il);
}

__global__ void tlas_expand_f64(int64_t n, const float4* __restrict__ hits, const float* __restrict__ rays,
                                const InstDev* __restrict__ inst, const BlasDev* __restrict__ blas, double* t,
                                int64_t* oinst, int64_t* oprim, double* u, double* v, double* nrm,
                                const uint32_t* __restrict__ st32, int64_t* __restrict__ st64,
                                const double* __restrict__ o64, const double* __restrict__ d64,
                                const double* __restrict__ tmin64, const double* __restrict__ tmax64, double tmin_s,
                                double tmax_s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 h0 = hits[2 * i], h1 = hits[2 * i + 1];
        const int ii = __float_as_int(h0.y), p = __float_as_int(h0.z);
        if (st32) { st64[2 * i] = st32[2 * i]; st64[2 * i + 1] = st32[2 * i + 1]; }
        if (ii < 0) {
            t[i] = -1.0; oinst[i] = -1; oprim[i] = -1; u[i] = -1.0; v[i] = -1.0;
            nrm[3 * i] = nrm[3 * i + 1] = nrm[3 * i + 2] = 0.0;
            continue;
        }
        const InstDev* I = inst + ii;
        const BlasDev B = blas[I->blas];
        double m[12];
        for (int k = 0; k < 12; ++k) m[k] = I->inv64[k];
        double ln[3];
        if (B.kind == 0) {
            ln[0] = B.lnormal[3 * p]; ln[1] = B.lnormal[3 * p + 1]; ln[2] = B.lnormal[3 * p + 2];
        } else {                                   // geometry.py:360-363 at the hit, local space
            const TraceRay r = load_ray(rays, i);
            double o[3], d[3];
            to_local_f64(m, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, o, d);
            const double* row = B.data + 4 * (int64_t)p;
            const double th = h0.x;
            for (int k = 0; k < 3; ++k) ln[k] = (o[k] + d[k] * th - row[k]) / row[3];
        }
        world_normal_f64(m, ln[0], ln[1], ln[2], nrm + 3 * i);
        double th = h0.x, uh = h0.w, vh = h1.x;
        if (B.kind == 0 && B.lrows && o64) {
            // the reference's own arithmetic: the float64 world ray to local space with the
            // float64 inverse (accel.py:804-809), then _tri_hit on the float64 local vertices
            double o[3], d[3], u2, v2;
            to_local_f64(m, o64[3 * i], o64[3 * i + 1], o64[3 * i + 2], d64[3 * i], d64[3 * i + 1], d64[3 * i + 2],
                         o, d);
            const double t2 = tri_hit_f64(o, d, tmin64 ? tmin64[i] : tmin_s, tmax64 ? tmax64[i] : tmax_s,
                                          B.lrows + 9 * (int64_t)p, u2, v2);
            const double hi_t = tmax64 ? tmax64[i] : tmax_s;
            if (t2 >= 0.0 && t2 < hi_t) {        // [t_min, t_max): accel.py:771-773, 815-817
                th = t2; uh = u2; vh = v2;
            } else if (t2 >= 0.0 || tri_hit_f64(o, d, 0.0, INFINITY, B.lrows + 9 * (int64_t)p, u2, v2) >= 0.0) {
                th = -1.0;                         // a float64 hit, outside [t_min, t_max]: a miss
            }
        }
        if (o64) {
            // the walk's fp32 window is the caller's rounded outward by a few ulps: a hit
            // outside the exact window is not the reference's hit
            const double lo_t = tmin64 ? tmin64[i] : tmin_s, hi_t = tmax64 ? tmax64[i] : tmax_s;
            if (th < lo_t || !(th < hi_t)) {
                t[i] = -1.0; oinst[i] = -1; oprim[i] = -1; u[i] = -1.0; v[i] = -1.0;
                nrm[3 * i] = nrm[3 * i + 1] = nrm[3 * i + 2] = 0.0;
                continue;
            }
        }
        t[i] = th; oinst[i] = ii; oprim[i] = p; u[i] = uh; v[i] = vh;
    }
}

// ---- device flatten (render a two-level scene through the flat LBVH path) ----
struct FlatInst {
    double m[12];             // instance matrix (world <- local), frame_to_matrix
    double inv[12];           // its inverse (normals, accel.py:843-847)
    const float* ltris;       // BLAS local vertices in prim order, (n_b, 9) fp32
    const double* lnormal;    // BLAS float64 local normals
    int64_t off;              // first flat id
    int inst;                 // instance index
    uint32_t mask;
    int material;
    int pad;
};

__device__ __forceinline__ double madd3(const double* r, double x, double y, double z, double t) {
    return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(r[0], x), __dmul_rn(r[1], y)), __dmul_rn(r[2], z)), t);
}

// one thread per flat triangle: world vertices (float64 in the host flatten's order,
// rounded to fp32), the reference-style world normal, ids, mask, material
__global__ void flatten_tris_kernel(const FlatInst* __restrict__ fi, int n_fi, int64_t n_tri, float* __restrict__ tris,
                                    float4* __restrict__ attr, int32_t* __restrict__ tinst,
                                    int32_t* __restrict__ tprim, uint32_t* __restrict__ tmask) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_tri; k += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = n_fi - 1;                    // last instance with off <= k
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (fi[mid].off <= k) lo = mid; else hi = mid - 1;
        }
        const FlatInst& F = fi[lo];
        const int64_t p = k - F.off;
        const float* v = F.ltris + 9 * p;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double x = v[3 * j], y = v[3 * j + 1], z = v[3 * j + 2];
            tris[9 * k + 3 * j + 0] = (float)madd3(F.m + 0, x, y, z, F.m[3]);
            tris[9 * k + 3 * j + 1] = (float)madd3(F.m + 4, x, y, z, F.m[7]);
            tris[9 * k + 3 * j + 2] = (float)madd3(F.m + 8, x, y, z, F.m[11]);
        }
        double wn[3];
        world_normal_f64(F.inv, F.lnormal[3 * p], F.lnormal[3 * p + 1], F.lnormal[3 * p + 2], wn);
        attr[k] = make_float4((float)wn[0], (float)wn[1], (float)wn[2], __int_as_float(F.material));
        tinst[k] = F.inst;
        tprim[k] = (int32_t)p;
        tmask[k] = F.mask;
    }
}

int tlas_view(rt_ctx* c, rt_tlas* T, TlasView& V) {
    V.tbvh4 = T->top->bvh4;
    V.ttris = T->top->tri_sorted;
    V.troot = T->top_root4;
    V.inst = T->d_inst;
    V.blas = T->d_blas;
    V.err = c->d_error;
    return RT_OK;
}

int read_root(rt_ctx* c, rt_scene* s, int& root4, int& height) {
    float4 n3;
    RT_CUDA_TRY(cudaMemcpyAsync(&n3, s->nodes + 3, sizeof n3, cudaMemcpyDeviceToHost, c->stream));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    memcpy(&height, &n3.z, 4);
    memcpy(&root4, &n3.w, 4);
    return RT_OK;
}

int upload_inst(rt_ctx* c, rt_tlas* T, const double* inv12) {
    for (int i = 0; i < T->n_inst; ++i) {
        InstDev& I = T->hinst[i];
        for (int k = 0; k < 12; ++k) {
            I.inv64[k] = inv12[12 * i + k];
            I.inv[k] = (float)inv12[12 * i + k];
        }
    }
    RT_CUDA_TRY(cudaMemcpyAsync(T->d_inst, T->hinst.data(), sizeof(InstDev) * T->n_inst, cudaMemcpyHostToDevice,
                                c->stream));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return RT_OK;
}

int build_top(rt_ctx* c, rt_tlas* T, const float* boxes6) {
    std::vector<float> tris(9 * (size_t)T->n_inst);
    for (int i = 0; i < T->n_inst; ++i) {
        const float* b = boxes6 + 6 * i;
        float* q = tris.data() + 9 * (size_t)i;
        q[0] = b[0]; q[1] = b[1]; q[2] = b[2];
        q[3] = b[3]; q[4] = b[4]; q[5] = b[5];
        q[6] = b[0]; q[7] = b[1]; q[8] = b[2];
    }
    int rc = rt_scene_set_vertices(c, T->top, tris.data());
    if (rc) return rc;
    rc = rt_bvh_build(c, T->top, 30, nullptr);
    if (rc) return rc;
    return read_root(c, T->top, T->top_root4, T->top_height);
}

}  // namespace

extern "C" {

int rt_scene_set_local_normals(rt_ctx* c, rt_scene* s, const double* n3) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && n3, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    if (!s->lnormal64) RT_CUDA_TRY(rt_alloc((void**)&s->lnormal64, sizeof(double) * 3 * (size_t)s->n, s->stream));
    RT_CUDA_TRY(cudaMemcpy(s->lnormal64, n3, sizeof(double) * 3 * (size_t)s->n, cudaMemcpyHostToDevice));
    return RT_OK;
}

int rt_scene_set_local_rows(rt_ctx* c, rt_scene* s, const double* rows9) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && rows9, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    if (!s->lrows64) RT_CUDA_TRY(rt_alloc((void**)&s->lrows64, sizeof(double) * 9 * (size_t)s->n, s->stream));
    RT_CUDA_TRY(cudaMemcpy(s->lrows64, rows9, sizeof(double) * 9 * (size_t)s->n, cudaMemcpyHostToDevice));
    return RT_OK;
}

int rt_scene_set_custom(rt_ctx* c, rt_scene* s, int32_t geom_type, int64_t data_offset) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && geom_type >= 0 && data_offset >= 0, "bad custom primitive description");
    s->custom = 1;
    s->geom_type = geom_type;
    s->data_offset = data_offset;
    return RT_OK;
}

int rt_tlas_create(rt_ctx* c, int32_t n_inst, rt_scene* const* inst_blas, const double* inv12, const float* boxes6,
                   const uint32_t* masks, rt_tlas** out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && out && n_inst >= 1 && inst_blas && inv12 && boxes6 && masks, "bad tlas arguments");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_tlas* T = new rt_tlas();
    T->n_inst = n_inst;
    std::map<rt_scene*, int> idx;
    for (int i = 0; i < n_inst; ++i) {
        rt_scene* b = inst_blas[i];
        if (!b || !b->built) {
            delete T;
            rt_set_error("instance %d references an unbuilt blas", i);
            return RT_EINVAL;
        }
        auto it = idx.find(b);
        if (it == idx.end()) {
            it = idx.emplace(b, (int)T->blas.size()).first;
            T->blas.push_back(b);
        }
        T->inst_blas.push_back(it->second);
    }
    // top level: an rt_scene over the instance boxes; flat id == instance, mask per prim
    std::vector<float> zeros(9 * (size_t)n_inst, 0.f), nz(3 * (size_t)n_inst, 0.f), mat(3, 0.f);
    std::vector<int32_t> ids(n_inst), prim(n_inst, 0), tmat(n_inst, 0);
    for (int i = 0; i < n_inst; ++i) ids[i] = i;
    int rc = rt_scene_create(c, n_inst, zeros.data(), nz.data(), ids.data(), prim.data(), masks, tmat.data(),
                             mat.data(), mat.data(), 1, &T->top);
    if (rc) { delete T; return rc; }
    T->hblas.resize(T->blas.size());
    T->d_data.assign(T->blas.size(), nullptr);
    T->max_height = 0;
    for (size_t b = 0; b < T->blas.size(); ++b) {
        rt_scene* s = T->blas[b];
        BlasDev& B = T->hblas[b];
        B.bvh4 = s->bvh4;
        B.tris = s->tri_sorted;
        B.lnormal = s->lnormal64;
        B.lrows = s->lrows64;
        B.data = nullptr;
        B.kind = s->custom ? 1 : 0;
        B.geom_type = s->custom ? s->geom_type : -1;
        if (!s->custom && !s->lnormal64) {
            rt_tlas_destroy(T);
            rt_set_error("triangle blas without local normals (rt_scene_set_local_normals)");
            return RT_EINVAL;
        }
        rc = read_root(c, s, B.root4, B.height);
        if (rc) { rt_tlas_destroy(T); return rc; }
        T->max_height = std::max(T->max_height, B.height);
    }
    T->hinst.resize(n_inst);
    for (int i = 0; i < n_inst; ++i) {
        T->hinst[i].mask = masks[i];
        T->hinst[i].blas = T->inst_blas[i];
        T->hinst[i].pad0 = T->hinst[i].pad1 = 0;
    }
    cudaError_t e1 = cudaMalloc(&T->d_blas, sizeof(BlasDev) * T->hblas.size());
    cudaError_t e2 = cudaMalloc(&T->d_inst, sizeof(InstDev) * n_inst);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
        rt_tlas_destroy(T);
        rt_set_error("cudaMalloc failed for the tlas tables");
        return RT_ENOMEM;
    }
    RT_CUDA_TRY(cudaMemcpy(T->d_blas, T->hblas.data(), sizeof(BlasDev) * T->hblas.size(), cudaMemcpyHostToDevice));
    rc = upload_inst(c, T, inv12);
    if (!rc) rc = build_top(c, T, boxes6);
    if (rc) { rt_tlas_destroy(T); return rc; }
    T->max_height = std::max(T->max_height, T->top_height);
    *out = T;
    return RT_OK;
}

int rt_tlas_update(rt_ctx* c, rt_tlas* T, const double* inv12, const float* boxes6) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && T && inv12 && boxes6, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    // BLAS refits may have changed their roots / heights (rebuilt LBVH)
    T->max_height = 0;
    for (size_t b = 0; b < T->blas.size(); ++b) {
        int rc = read_root(c, T->blas[b], T->hblas[b].root4, T->hblas[b].height);
        if (rc) return rc;
        T->hblas[b].bvh4 = T->blas[b]->bvh4;
        T->hblas[b].tris = T->blas[b]->tri_sorted;
        T->hblas[b].lrows = T->blas[b]->lrows64;
        T->max_height = std::max(T->max_height, T->hblas[b].height);
    }
    RT_CUDA_TRY(cudaMemcpy(T->d_blas, T->hblas.data(), sizeof(BlasDev) * T->hblas.size(), cudaMemcpyHostToDevice));
    int rc = upload_inst(c, T, inv12);
    if (rc) return rc;
    rc = build_top(c, T, boxes6);
    if (rc) return rc;
    T->max_height = std::max(T->max_height, T->top_height);
    return RT_OK;
}

int rt_tlas_set_custom_data(rt_ctx* c, rt_tlas* T, int32_t geom_type, int64_t n_rows, const double* rows4) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && T && n_rows >= 0 && (n_rows == 0 || rows4), "bad custom data");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    bool changed = false;
    for (size_t b = 0; b < T->blas.size(); ++b) {
        rt_scene* s = T->blas[b];
        if (!s->custom || s->geom_type != geom_type) continue;
        if (T->d_data[b]) cudaFree(T->d_data[b]);
        T->d_data[b] = nullptr;
        T->hblas[b].data = nullptr;
        changed = true;
        if (n_rows == 0) continue;                       // unregister
        if (s->data_offset + s->n > n_rows) {
            rt_set_error("custom data has %lld rows, blas needs rows [%lld, %lld)", (long long)n_rows,
                         (long long)s->data_offset, (long long)(s->data_offset + s->n));
            return RT_EINVAL;
        }
        RT_CUDA_TRY(cudaMalloc(&T->d_data[b], sizeof(double) * 4 * (size_t)s->n));
        RT_CUDA_TRY(cudaMemcpy(T->d_data[b], rows4 + 4 * s->data_offset, sizeof(double) * 4 * (size_t)s->n,
                               cudaMemcpyHostToDevice));
        T->hblas[b].data = T->d_data[b];
    }
    if (changed)
        RT_CUDA_TRY(cudaMemcpy(T->d_blas, T->hblas.data(), sizeof(BlasDev) * T->hblas.size(),
                               cudaMemcpyHostToDevice));
    return RT_OK;
}

void rt_tlas_destroy(rt_tlas* T) {
    if (!T) return;
    if (T->top) rt_scene_destroy(T->top);
    if (T->d_blas) cudaFree(T->d_blas);
    if (T->d_inst) cudaFree(T->d_inst);
    for (double* p : T->d_data)
        if (p) cudaFree(p);
    delete T;
}

// Flat single-level scene from a two-level one, built on the device: the triangle
// instances (all before any custom instance, so flat ids stay in (instance, prim)
// order) are transformed by flatten_tris_kernel; custom primitives are appended from
// host rows like compile_scene's spheres.  *io: NULL -> a new scene; else a scene of
// the same size is refilled in place (after refits / frame edits).  Built with LBVH-bits.
int rt_tlas_flatten(rt_ctx* c, rt_tlas* T, const double* mat12, const int32_t* inst_material, const float* mat_color,
                    const float* mat_emissive, int32_t n_mat, int32_t n_custom, const float* custom_boxes9,
                    const double* custom_rows16, const int32_t* custom_inst, const int32_t* custom_prim,
                    int32_t bits, rt_scene** io) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && T && mat12 && inst_material && mat_color && mat_emissive && io, "NULL argument");
    RT_CHECK_ARG(n_custom >= 0 && (n_custom == 0 || (custom_boxes9 && custom_rows16 && custom_inst && custom_prim)),
                 "bad custom primitive rows");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    std::vector<FlatInst> fi;
    int64_t n_tri = 0;
    bool seen_custom = false;
    for (int i = 0; i < T->n_inst; ++i) {
        rt_scene* b = T->blas[T->inst_blas[i]];
        if (b->custom) { seen_custom = true; continue; }
        if (seen_custom) {
            rt_set_error("flatten needs every triangle instance before the custom-primitive instances");
            return RT_EINVAL;
        }
        RT_CHECK_ARG(inst_material[i] >= 0 && inst_material[i] < n_mat, "instance material out of range");
        FlatInst f;
        for (int k = 0; k < 12; ++k) { f.m[k] = mat12[12 * i + k]; f.inv[k] = T->hinst[i].inv64[k]; }
        f.ltris = b->tris;
        f.lnormal = b->lnormal64;
        f.off = n_tri;
        f.inst = i;
        f.mask = T->hinst[i].mask;
        f.material = inst_material[i];
        f.pad = 0;
        fi.push_back(f);
        n_tri += b->n;
    }
    const int64_t n = n_tri + n_custom;
    RT_CHECK_ARG(n >= 1, "cannot build over zero primitives");
    rt_scene* s = *io;
    if (s && (s->n != n || s->n_mat != n_mat)) {
        rt_set_error("flatten target has %lld primitives / %d materials, need %lld / %d", (long long)s->n, s->n_mat,
                     (long long)n, n_mat);
        return RT_EINVAL;
    }
    const bool fresh = s == nullptr;
    if (fresh) {
        int rc = rt_scene_alloc(c, n, n_mat, &s);
        if (rc) return rc;
    }
    auto bail = [&](int rc) { if (fresh) rt_scene_destroy(s); return rc; };
    FlatInst* d_fi = nullptr;
    cudaError_t e = cudaSuccess;
    if (!fi.empty()) {
        if ((e = cudaMalloc(&d_fi, sizeof(FlatInst) * fi.size())) ||
            (e = cudaMemcpy(d_fi, fi.data(), sizeof(FlatInst) * fi.size(), cudaMemcpyHostToDevice))) {
            if (d_fi) cudaFree(d_fi);
            rt_set_error("flatten upload: %s", cudaGetErrorString(e));
            return bail(RT_ECUDA);
        }
        flatten_tris_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(d_fi, (int)fi.size(), n_tri, s->tris, s->tri_attr,
                                                                    s->tri_inst, s->tri_prim, s->tri_mask);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && n_custom) {
        std::vector<float4> attr(n_custom);
        std::vector<uint32_t> mk(n_custom);
        for (int k = 0; k < n_custom; ++k) {
            const int i = custom_inst[k];
            float mf;
            memcpy(&mf, &inst_material[i], 4);
            attr[k] = make_float4(0.f, 0.f, 0.f, mf);
            mk[k] = T->hinst[i].mask;
        }
        cudaStream_t st = c->stream;
        if (!(e = cudaMemcpyAsync(s->tris + 9 * n_tri, custom_boxes9, sizeof(float) * 9 * n_custom,
                                  cudaMemcpyHostToDevice, st)) &&
            !(e = cudaMemcpyAsync(s->tri_attr + n_tri, attr.data(), sizeof(float4) * n_custom, cudaMemcpyHostToDevice,
                                  st)) &&
            !(e = cudaMemcpyAsync(s->tri_inst + n_tri, custom_inst, 4 * n_custom, cudaMemcpyHostToDevice, st)) &&
            !(e = cudaMemcpyAsync(s->tri_prim + n_tri, custom_prim, 4 * n_custom, cudaMemcpyHostToDevice, st)) &&
            !(e = cudaMemcpyAsync(s->tri_mask + n_tri, mk.data(), 4 * n_custom, cudaMemcpyHostToDevice, st)))
            e = cudaStreamSynchronize(st);
    }
    if (d_fi) {
        cudaError_t e2 = cudaStreamSynchronize(c->stream);
        cudaFree(d_fi);
        if (e == cudaSuccess) e = e2;
    }
    if (e != cudaSuccess) {
        rt_set_error("flatten: %s", cudaGetErrorString(e));
        return bail(RT_ECUDA);
    }
    s->mask_uniform = 1;
    s->mask_value = T->hinst[0].mask;
    for (int i = 1; i < T->n_inst; ++i) s->mask_uniform &= T->hinst[i].mask == s->mask_value;
    int rc = rt_scene_set_materials(c, s, mat_color, mat_emissive);
    if (!rc) rc = rt_scene_set_spheres(c, s, n_custom, n_custom ? custom_rows16 : nullptr);
    if (!rc) rc = rt_bvh_build(c, s, bits, nullptr);
    if (rc) return bail(rc);
    *io = s;
    return RT_OK;
}

int rt_tlas_info(rt_ctx* c, rt_tlas* T, float* root6, int32_t* height) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && T, "NULL argument");
    return rt_bvh_info(c, T->top, root6, height, nullptr);
}

// accel.py:1128-1156 closest_hit_batch over a two-level structure (host float64 rays,
// hostio.cuh pipeline)
int rt_tlas_closest_host(rt_ctx* c, rt_tlas* T, int64_t n, const double* o, const double* d, const double* tmin,
                         const double* tmax, double tmin_s, double tmax_s, uint32_t ray_mask, double* t,
                         int64_t* inst, int64_t* prim, double* u, double* v, double* nrm, int64_t* stats) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && T, "NULL argument");
    RT_CHECK_ARG(n >= 0, "negative ray count");
    RT_CHECK_ARG(n == 0 || (o && d && t && inst && prim && u && v && nrm), "NULL ray or output buffer");
    if (n == 0) return RT_OK;
    RT_CUDA_TRY(cudaSetDevice(c->device));
    TlasView V;
    tlas_view(c, T, V);
    const HostIo in{o, d, tmin, tmax, tmin_s, tmax_s};
    // hits: 2 float4 + stats u32 pair; out: t, inst, prim, u, v, normal, stats i64 pair
    auto kernels = [&](const IoSlot& S, int64_t m) -> int {
        float4* hits = (float4*)S.hits;
        uint32_t* st = stats ? (uint32_t*)((char*)S.hits + 32 * m) : nullptr;
        RT_CUDA_TRY(cudaMemsetAsync(c->d_counter, 0, sizeof(unsigned), c->stream));
        int bps = 0;
        if (stats) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, tlas_closest_kernel<true>, TL_THREADS, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, tlas_closest_kernel<false>, TL_THREADS, 0);
        if (bps < 1) bps = 1;
        const int64_t grid = std::min<int64_t>((int64_t)c->num_sms * bps, (m + TL_THREADS - 1) / TL_THREADS);
        if (stats)
            tlas_closest_kernel<true><<<(unsigned)grid, TL_THREADS, 0, c->stream>>>(
                V, T->max_height, m, S.rays, hits, ray_mask, st, c->d_counter);
        else
            tlas_closest_kernel<false><<<(unsigned)grid, TL_THREADS, 0, c->stream>>>(
                V, T->max_height, m, S.rays, hits, ray_mask, nullptr, c->d_counter);
        RT_CUDA_TRY(cudaGetLastError());
        char* O = (char*)S.out;
        tlas_expand_f64<<<c->num_sms * 4, 256, 0, c->stream>>>(
            m, hits, S.rays, T->d_inst, T->d_blas, (double*)O, (int64_t*)(O + 8 * m), (int64_t*)(O + 16 * m),
            (double*)(O + 24 * m), (double*)(O + 32 * m), (double*)(O + 40 * m), st, (int64_t*)(O + 64 * m), S.o, S.d,
            tmin ? S.tmin : nullptr, tmax ? S.tmax : nullptr, tmin_s, tmax_s);
        RT_CUDA_TRY(cudaGetLastError());
        return RT_OK;
    };
    auto download = [&](const IoSlot& S, int64_t b, int64_t m, cudaStream_t so) -> int {
        const char* O = (const char*)S.out;
        RT_CUDA_TRY(cudaMemcpyAsync(t + b, O, 8 * m, cudaMemcpyDeviceToHost, so));
        RT_CUDA_TRY(cudaMemcpyAsync(inst + b, O + 8 * m, 8 * m, cudaMemcpyDeviceToHost, so));
        RT_CUDA_TRY(cudaMemcpyAsync(prim + b, O + 16 * m, 8 * m, cudaMemcpyDeviceToHost, so));
        RT_CUDA_TRY(cudaMemcpyAsync(u + b, O + 24 * m, 8 * m, cudaMemcpyDeviceToHost, so));
        RT_CUDA_TRY(cudaMemcpyAsync(v + b, O + 32 * m, 8 * m, cudaMemcpyDeviceToHost, so));
        RT_CUDA_TRY(cudaMemcpyAsync(nrm + 3 * b, O + 40 * m, 24 * m, cudaMemcpyDeviceToHost, so));
        if (stats) RT_CUDA_TRY(cudaMemcpyAsync(stats + 2 * b, O + 64 * m, 16 * m, cudaMemcpyDeviceToHost, so));
        return RT_OK;
    };
    int rc = rt_io_run(c, n, in, 40, 80, kernels, download);
    if (rc) return rc;
    return rt_check_device_error(c);
}

// accel.py:1159-1174 any_hit_batch over a two-level structure
int rt_tlas_any_host(rt_ctx* c, rt_tlas* T, int64_t n, const double* o, const double* d, const double* tmin,
                     const double* tmax, double tmin_s, double tmax_s, uint32_t ray_mask, uint8_t* out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && T, "NULL argument");
    RT_CHECK_ARG(n >= 0, "negative ray count");
    RT_CHECK_ARG(n == 0 || (o && d && out), "NULL ray or output buffer");
    if (n == 0) return RT_OK;
    RT_CUDA_TRY(cudaSetDevice(c->device));
    TlasView V;
    tlas_view(c, T, V);
    const HostIo in{o, d, tmin, tmax, tmin_s, tmax_s};
    auto kernels = [&](const IoSlot& S, int64_t m) -> int {
        RT_CUDA_TRY(cudaMemsetAsync(c->d_counter, 0, sizeof(unsigned), c->stream));
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, tlas_any_kernel, TL_THREADS, 0);
        if (bps < 1) bps = 1;
        const int64_t grid = std::min<int64_t>((int64_t)c->num_sms * bps, (m + TL_THREADS - 1) / TL_THREADS);
        tlas_any_kernel<<<(unsigned)grid, TL_THREADS, 0, c->stream>>>(V, T->max_height, m, S.rays,
                                                                      (uint8_t*)S.out, ray_mask, c->d_counter);
        RT_CUDA_TRY(cudaGetLastError());
        return RT_OK;
    };
    auto download = [&](const IoSlot& S, int64_t b, int64_t m, cudaStream_t so) -> int {
        RT_CUDA_TRY(cudaMemcpyAsync(out + b, S.out, m, cudaMemcpyDeviceToHost, so));
        return RT_OK;
    };
    int rc = rt_io_run(c, n, in, 0, 1, kernels, download);
    if (rc) return rc;
    return rt_check_device_error(c);
}

}  // extern "C"
