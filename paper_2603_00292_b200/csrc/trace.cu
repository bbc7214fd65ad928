// trace.cu -- K6: persistent-thread closest-hit kernel over a ray buffer, plus
// the f64 <-> f32 packing kernels behind rt_closest_hit_host (the reference's
// closest_hit_batch dtypes, accel.py:1128-1156).
#include "hostio.cuh"
#include "traverse.cuh"

namespace {

constexpr int TRACE_THREADS = 128;
#ifndef RT_SMEM_STACK
#define RT_SMEM_STACK 0
#endif

// One warp fetches 32 rays at a time from a global counter (one atomicAdd per
// warp), every lane runs the while-while traversal, then the warp fetches again.
template <bool STATS, bool SPH>
__global__ void __launch_bounds__(TRACE_THREADS, 8) trace_closest_kernel(
    const float4* __restrict__ nodes, const float4* __restrict__ bvh4, const float4* __restrict__ tris, int64_t n,
    const float* __restrict__ rays, float4* __restrict__ hits, uint32_t ray_mask, uint32_t* __restrict__ stats,
    unsigned int* counter, int* err, const SphereView sv) {
    const int height = __float_as_int(__ldg(nodes + 3).z);   // root height == stack bound
    const int root4 = __float_as_int(__ldg(nodes + 3).w);    // BVH4 root (split position)
    if (height + 1 > RT_STACK) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(err, RT_EDEPTH);
        return;
    }
    int2 stack[RT_STACK4];
#if RT_SMEM_STACK
    __shared__ int2 s_stack[RT_SMEM_STACK * TRACE_THREADS];
    const SmemStack<RT_SMEM_STACK, TRACE_THREADS> walk_stack{s_stack + threadIdx.x, stack};
#else
    const LocalStack walk_stack{stack};
#endif
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(counter, 32u);
        base = __shfl_sync(RT_FULL, base, 0);
        if ((int64_t)base >= n) break;
        int64_t i = (int64_t)base + lane;
        if (i < n) {
            TraceRay r = load_ray(rays, i);
            RayPre R;
            ray_setup(R, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, r.tmin);
            uint32_t nt = 0, nv = 0;
            HitRec h = trace_ray4<STATS, SPH>(bvh4, root4, tris, R, r.tmax, ray_mask, walk_stack, nt, nv, sv);
            hits[i] = make_float4(h.t, __int_as_float(h.id), h.u, h.v);
            if (STATS) reinterpret_cast<uint2*>(stats)[i] = make_uint2(nt, nv);
        }
    }
}

// any-hit over a ray buffer (same persistent warp fetch as the closest-hit kernel)
template <bool SPH>
__global__ void __launch_bounds__(TRACE_THREADS, 8) trace_any_kernel(
    const float4* __restrict__ nodes, const float4* __restrict__ bvh4, const float4* __restrict__ tris, int64_t n,
    const float* __restrict__ rays, uint8_t* __restrict__ out, uint32_t ray_mask, unsigned int* counter, int* err,
    const SphereView sv) {
    const int height = __float_as_int(__ldg(nodes + 3).z);
    const int root4 = __float_as_int(__ldg(nodes + 3).w);
    if (height + 1 > RT_STACK) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(err, RT_EDEPTH);
        return;
    }
    int stack[RT_STACK4];
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(counter, 32u);
        base = __shfl_sync(RT_FULL, base, 0);
        if ((int64_t)base >= n) break;
        int64_t i = (int64_t)base + lane;
        if (i < n) {
            TraceRay r = load_ray(rays, i);
            RayPre R;
            ray_setup(R, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, r.tmin);
            out[i] = trace_any4<SPH>(bvh4, root4, tris, R, r.tmax, ray_mask, stack, sv) ? 1 : 0;
        }
    }
}

// float64 rays -> the fp32 trace layout; t ranges per ray (arrays) or broadcast (scalars)
__global__ void pack_rays_f64(int64_t n, const double* __restrict__ o, const double* __restrict__ d,
                              const double* __restrict__ tmin, const double* __restrict__ tmax, double tmin_s,
                              double tmax_s, float4* __restrict__ rays) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double tn = tmin ? tmin[i] : tmin_s;
        const double tm = tmax ? tmax[i] : tmax_s;
        // the fp32 window contains the float64 one with a few ulps to spare (t_min rounded
        // down, t_max up, then widened by 2^-21 relative: the fp32 triangle t carries a few
        // ulps of error), so the walk never loses a hit the reference accepts;
        // expand_hits_f64 re-checks the exact window
        float tn32 = __double2float_rd(tn), tm32 = tm > 3.0e38 ? INFINITY : __double2float_ru(tm);
        tn32 = tn32 > 0.f ? __fmul_rd(tn32, 1.0f - 0x1p-21f) : __fmul_rd(tn32, 1.0f + 0x1p-21f);
        tm32 = tm32 > 0.f ? __fmul_ru(tm32, 1.0f + 0x1p-21f) : __fmul_ru(tm32, 1.0f - 0x1p-21f);
        rays[2 * i] = make_float4((float)o[3 * i], (float)o[3 * i + 1], (float)o[3 * i + 2], tn32);
        rays[2 * i + 1] = make_float4((float)d[3 * i], (float)d[3 * i + 1], (float)d[3 * i + 2], tm32);
    }
}

// hit (t, id, u, v) -> the reference's per-ray outputs (float64 / int64),
// world normal from the per-triangle reference-style normal, or
// the sphere's at the hit point (rays needed only then).  With the caller's float64
// rays (host query API), a triangle hit's (t, u, v) are recomputed in float64 with the
// reference's own formula on that triangle: bit-identical to the reference whenever
// it hits the same triangle with the same (fp32-valued) world vertices; the fp32
// values stay if the float64 test rejects the pair (edge / grazing cases).
__global__ void expand_hits_f64(int64_t n, const float4* __restrict__ hits, const float4* __restrict__ attr,
                                const int32_t* __restrict__ tri_inst, const int32_t* __restrict__ tri_prim,
                                double* t, int64_t* inst, int64_t* prim, double* u, double* v, double* nrm,
                                const float* __restrict__ rays, const SphereView sv,
                                const uint32_t* __restrict__ st32, int64_t* __restrict__ st64,
                                const float* __restrict__ wtris, const double* __restrict__ o64,
                                const double* __restrict__ d64, const double* __restrict__ tmin64,
                                const double* __restrict__ tmax64, double tmin_s, double tmax_s,
                                const double* __restrict__ wn64, const double* __restrict__ inv64,
                                const double* __restrict__ lrows64) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float4 h = hits[i];
        int id = __float_as_int(h.y);
        if (id < 0) {
            t[i] = -1.0; inst[i] = -1; prim[i] = -1; u[i] = -1.0; v[i] = -1.0;
            nrm[3 * i] = 0.0; nrm[3 * i + 1] = 0.0; nrm[3 * i + 2] = 0.0;
        } else {
            float4 a = attr[id];
            double th = h.x, uh = h.z, vh = h.w;
            if (o64 && id < sv.base) {
                double o[3] = {o64[3 * i], o64[3 * i + 1], o64[3 * i + 2]};
                double d[3] = {d64[3 * i], d64[3 * i + 1], d64[3 * i + 2]};
                double u2, v2, t2;
                const double lo_t = tmin64 ? tmin64[i] : tmin_s, hi_t = tmax64 ? tmax64[i] : tmax_s;
                const double* row;
                double ol[3], dl[3];
                if (inv64 && lrows64) {
                    // exactly the reference's path: the ray to the instance's local space with
                    // its float64 inverse (accel.py:804-809), _tri_hit on the local vertices
                    double m[12];
                    const int ins = tri_inst[id];
#pragma unroll
                    for (int k = 0; k < 12; ++k) m[k] = inv64[12 * (int64_t)ins + k];
                    to_local_f64(m, o[0], o[1], o[2], d[0], d[1], d[2], ol, dl);
                    row = lrows64 + 9 * (int64_t)id;
                } else {
                    for (int k = 0; k < 3; ++k) { ol[k] = o[k]; dl[k] = d[k]; }
                    row = nullptr;
                }
                if (row) t2 = tri_hit_f64(ol, dl, lo_t, hi_t, row, u2, v2);
                else t2 = tri_hit_f64(o, d, lo_t, hi_t, wtris + 9 * (int64_t)id, u2, v2);
                // a hit exactly at t_max is not taken by the reference's scene-level rule
                // (t < best_t, or t == best_t with a lower instance than best_inst = -1;
                // accel.py:771-773, 815-817): its closest-hit window is [t_min, t_max)
                if (t2 >= 0.0 && !(t2 < hi_t)) t2 = -1.0;
                if (t2 >= 0.0) {
                    th = t2; uh = u2; vh = v2;
                } else {
                    // rejected: outside [t_min, t_max] (the fp32 walk's window is the caller's
                    // rounded outward by a few ulps) -> not the reference's hit, a miss; or a
                    // geometric edge / grazing case of the float64 test -> the fp32 values stay
                    const double t3 = row ? tri_hit_f64(ol, dl, 0.0, INFINITY, row, u2, v2)
                                          : tri_hit_f64(o, d, 0.0, INFINITY, wtris + 9 * (int64_t)id, u2, v2);
                    if (t3 >= 0.0 || th < lo_t || !(th < hi_t)) id = -1;
                }
            } else if (o64) {                                    // spheres: the exact window
                if (th < (tmin64 ? tmin64[i] : tmin_s) || !(th < (tmax64 ? tmax64[i] : tmax_s))) id = -1;
            }
            if (id < 0) {
                t[i] = -1.0; inst[i] = -1; prim[i] = -1; u[i] = -1.0; v[i] = -1.0;
                nrm[3 * i] = 0.0; nrm[3 * i + 1] = 0.0; nrm[3 * i + 2] = 0.0;
                if (st64) { st64[2 * i] = st32[2 * i]; st64[2 * i + 1] = st32[2 * i + 1]; }
                continue;
            }
            t[i] = th; inst[i] = tri_inst[id]; prim[i] = tri_prim[id]; u[i] = uh; v[i] = vh;
            if (id >= sv.base) {
                const TraceRay r = load_ray(rays, i);
                const float3 w = sphere_normal(sv.rows + 16 * (int64_t)(id - sv.base), r.ox, r.oy, r.oz, r.dx, r.dy,
                                               r.dz, h.x);
                a.x = w.x; a.y = w.y; a.z = w.z;
                nrm[3 * i] = a.x; nrm[3 * i + 1] = a.y; nrm[3 * i + 2] = a.z;
            } else if (wn64) {            // the reference-style float64 world normal itself
                nrm[3 * i] = wn64[3 * id]; nrm[3 * i + 1] = wn64[3 * id + 1]; nrm[3 * i + 2] = wn64[3 * id + 2];
            } else {
                nrm[3 * i] = a.x; nrm[3 * i + 1] = a.y; nrm[3 * i + 2] = a.z;
            }
        }
        if (st64) { st64[2 * i] = st32[2 * i]; st64[2 * i + 1] = st32[2 * i + 1]; }
    }
}

}  // namespace

int rt_trace_impl(rt_ctx* ctx, rt_scene* s, int64_t n, const float* rays, float4* hits, uint32_t mask,
                  uint32_t* stats, int custom_mode) {
    if (n <= 0) return RT_OK;
    if ((n + 64) > 0xFFFFFFFFll) {
        rt_set_error("at most 2^32 - 65 rays per trace call (got %lld)", (long long)n);
        return RT_EINVAL;
    }
    cudaStream_t st = ctx->stream;
    RT_CUDA_TRY(cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned int), st));
    const SphereView sv = rt_sphere_view(ctx, s, custom_mode);
    auto launch = [&](auto kern, uint32_t* st_ptr) {
        int blocks_per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, TRACE_THREADS, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        int64_t want = (n + TRACE_THREADS - 1) / TRACE_THREADS;
        int64_t grid = (int64_t)ctx->num_sms * blocks_per_sm;
        if (grid > want) grid = want;
        kern<<<(unsigned)grid, TRACE_THREADS, 0, st>>>(s->nodes, s->bvh4, s->tri_sorted, n, rays, hits, mask, st_ptr,
                                                       ctx->d_counter, ctx->d_error, sv);
    };
    const bool sph = s->n_spheres > 0;
    if (stats) {
        if (sph) launch(trace_closest_kernel<true, true>, stats);
        else launch(trace_closest_kernel<true, false>, stats);
    } else {
        if (sph) launch(trace_closest_kernel<false, true>, nullptr);
        else launch(trace_closest_kernel<false, false>, nullptr);
    }
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

int rt_trace_any_impl(rt_ctx* ctx, rt_scene* s, int64_t n, const float* rays, uint8_t* out, uint32_t mask,
                      int custom_mode) {
    if (n <= 0) return RT_OK;
    if ((n + 64) > 0xFFFFFFFFll) {
        rt_set_error("at most 2^32 - 65 rays per trace call (got %lld)", (long long)n);
        return RT_EINVAL;
    }
    cudaStream_t st = ctx->stream;
    RT_CUDA_TRY(cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned int), st));
    const SphereView sv = rt_sphere_view(ctx, s, custom_mode);
    auto launch = [&](auto kern) {
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, TRACE_THREADS, 0);
        if (bps < 1) bps = 1;
        int64_t want = (n + TRACE_THREADS - 1) / TRACE_THREADS;
        int64_t grid = (int64_t)ctx->num_sms * bps;
        if (grid > want) grid = want;
        kern<<<(unsigned)grid, TRACE_THREADS, 0, st>>>(s->nodes, s->bvh4, s->tri_sorted, n, rays, out, mask,
                                                       ctx->d_counter, ctx->d_error, sv);
    };
    if (s->n_spheres > 0) launch(trace_any_kernel<true>);
    else launch(trace_any_kernel<false>);
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

int rt_pack_rays_f64(rt_ctx* ctx, int64_t n, const double* o, const double* d, const double* tmin,
                     const double* tmax, float* rays) {
    int grid = ctx->num_sms * 8;
    pack_rays_f64<<<grid, 256, 0, ctx->stream>>>(n, o, d, tmin, tmax, 0.0, 0.0, reinterpret_cast<float4*>(rays));
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

int rt_pack_rays_io(rt_ctx* ctx, int64_t n, const IoSlot& s, bool per_ray_tmin, bool per_ray_tmax, double tmin_s,
                    double tmax_s) {
    int grid = ctx->num_sms * 8;
    pack_rays_f64<<<grid, 256, 0, ctx->stream>>>(n, s.o, s.d, per_ray_tmin ? s.tmin : nullptr,
                                                 per_ray_tmax ? s.tmax : nullptr, tmin_s, tmax_s,
                                                 reinterpret_cast<float4*>(s.rays));
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

int rt_io_streams(rt_ctx* c) {
    if (c->io_in) return RT_OK;
    RT_CUDA_TRY(cudaStreamCreateWithFlags(&c->io_in, cudaStreamNonBlocking));
    RT_CUDA_TRY(cudaStreamCreateWithFlags(&c->io_out, cudaStreamNonBlocking));
    for (int k = 0; k < 9; ++k) RT_CUDA_TRY(cudaEventCreateWithFlags(&c->io_ev[k], cudaEventDisableTiming));
    return RT_OK;
}

int rt_io_ensure(rt_ctx* c, int64_t chunk, size_t hit_bytes, size_t out_bytes, IoSlot slots[2]) {
    // per ray and slot: o 24, d 24, tmin 8, tmax 8, rays 32, hits, out (each region 256-B aligned)
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t m = (size_t)chunk;
    const size_t per_slot = al(24 * m) * 2 + al(8 * m) * 2 + al(32 * m) + al(hit_bytes * m + 16) + al(out_bytes * m);
    const size_t need = 2 * per_slot;
    if (c->d_io_bytes < need) {
        if (c->d_io) cudaFree(c->d_io);
        c->d_io = nullptr;
        c->d_io_bytes = 0;
        RT_CUDA_TRY(cudaMalloc(&c->d_io, need));
        c->d_io_bytes = need;
    }
    char* p = (char*)c->d_io;
    for (int k = 0; k < 2; ++k) {
        slots[k].o = (double*)p; p += al(24 * m);
        slots[k].d = (double*)p; p += al(24 * m);
        slots[k].tmin = (double*)p; p += al(8 * m);
        slots[k].tmax = (double*)p; p += al(8 * m);
        slots[k].rays = (float*)p; p += al(32 * m);
        slots[k].hits = p; p += al(hit_bytes * m + 16);
        slots[k].out = p; p += al(out_bytes * m);
    }
    return RT_OK;
}

int rt_expand_hits_f64(rt_ctx* ctx, rt_scene* s, int64_t n, const float4* hits, double* t, int64_t* inst,
                       int64_t* prim, double* u, double* v, double* nrm, const float* rays, const uint32_t* st32,
                       int64_t* st64, const double* o64, const double* d64, const double* tmin64,
                       const double* tmax64, double tmin_s, double tmax_s) {
    int grid = ctx->num_sms * 8;
    expand_hits_f64<<<grid, 256, 0, ctx->stream>>>(n, hits, s->tri_attr, s->tri_inst, s->tri_prim, t, inst, prim,
                                                    u, v, nrm, rays, rt_sphere_view(ctx, s, 0), st32,
                                                    st32 ? st64 : nullptr, s->tris, o64, d64, tmin64, tmax64, tmin_s,
                                                    tmax_s, s->wnormal64, s->inst_inv64, s->lrows64);
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}
