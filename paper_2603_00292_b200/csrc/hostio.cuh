// hostio.cuh -- the host-buffer entry points' transfer pipeline (closest_hit_batch /
// any_hit_batch with the reference's float64 / int64 host dtypes).
//
// Rays are processed in chunks through two device slots on three streams:
//   copy-in stream   H2D of chunk k's float64 origins / directions (/ t ranges)
//   context stream   pack to fp32 rays -> trace -> expand to the float64 outputs
//   copy-out stream  D2H of chunk k's outputs
// so chunk k+1's upload, chunk k's kernels and chunk k-1's download overlap
// (the two copy engines run H2D and D2H concurrently).  With pinned host buffers
// every copy is a full-rate async DMA; pageable buffers still work (the driver
// stages them synchronously).  Scalar t_min / t_max (the reference's default
// broadcast) are passed by value instead of as per-ray arrays.
#pragma once
#include <algorithm>
#include <vector>

#include "rt_common.cuh"

// Slot size: n / RT_IO_CHUNKS rays, clamped to [64K, 512K].  4 chunks: enough overlap;
// more cost more in per-copy / per-launch overhead than they save in pipeline fill and
// drain (config 2 e2e: 16 -> 436, 8 -> 485, 4 -> 490 Mrays/s).
#ifndef RT_IO_CHUNKS
#define RT_IO_CHUNKS 4
#endif
// Chunk sizes grow from RT_IO_FIRST rays (doubling) to the slot size, so the first
// download starts early (config-2 closest_hit_batch 3.63 -> 3.45 ms; first chunk 64K: 3.49)
#ifndef RT_IO_GEOMETRIC
#define RT_IO_GEOMETRIC 1
#endif
#ifndef RT_IO_FIRST
#define RT_IO_FIRST (1 << 17)
#endif

struct HostIo {
    const double* o;
    const double* d;
    const double* tmin;     // nullable: use tmin_s
    const double* tmax;     // nullable: use tmax_s
    double tmin_s, tmax_s;
};

// one slot of device staging
struct IoSlot {
    double* o;
    double* d;
    double* tmin;
    double* tmax;
    float* rays;
    void* hits;
    void* out;              // expand output area (layout owned by the caller)
};

int rt_io_ensure(rt_ctx* c, int64_t chunk, size_t hit_bytes, size_t out_bytes, IoSlot slots[2]);
int rt_io_streams(rt_ctx* c);
int rt_pack_rays_io(rt_ctx* ctx, int64_t n, const IoSlot& s, bool per_ray_tmin, bool per_ray_tmax, double tmin_s,
                    double tmax_s);

// Generic pipeline.  kernels(slot, m): enqueue pack/trace/expand for m rays of the
// slot on c->stream (pack is done here).  download(slot, b, m): enqueue the D2H of
// chunk [b, b+m) on the stream passed.  Returns after everything completed.
template <class Kernels, class Download>
int rt_io_run(rt_ctx* c, int64_t n, const HostIo& in, size_t hit_bytes, size_t out_bytes, Kernels&& kernels,
              Download&& download) {
    if (n <= 0) return RT_OK;
    int rc = rt_io_streams(c);
    if (rc) return rc;
    int64_t chunk = std::max<int64_t>(1 << 16, std::min<int64_t>(1 << 19, (n + RT_IO_CHUNKS - 1) / RT_IO_CHUNKS));
    chunk = std::min(chunk, n);
#if RT_IO_GEOMETRIC
    int64_t first = std::min<int64_t>(chunk, RT_IO_FIRST);
#endif
    IoSlot slots[2];
    rc = rt_io_ensure(c, chunk, hit_bytes, out_bytes, slots);
    if (rc) return rc;
    cudaStream_t sc = c->stream, si = c->io_in, so = c->io_out;
    // the staging slots are free (every earlier call synchronised its streams), so the
    // first uploads overlap whatever still runs on the context stream (e.g. a rebuild);
    // the kernels themselves queue behind it on that stream
    cudaEvent_t* in_ready = c->io_ev;          // [2]
    cudaEvent_t* in_free = c->io_ev + 2;       // [2]
    cudaEvent_t* out_free = c->io_ev + 4;      // [2]
    int64_t k = 0;
#if RT_IO_GEOMETRIC
    int64_t step = first;
    for (int64_t b = 0; b < n; b += step, step = std::min(chunk, 2 * step), ++k) {
        const int64_t m = std::min(step, n - b);
#else
    for (int64_t b = 0; b < n; b += chunk, ++k) {
        const int64_t m = std::min(chunk, n - b);
#endif
        const int s = (int)(k & 1);
        const IoSlot& S = slots[s];
        if (k >= 2) RT_CUDA_TRY(cudaStreamWaitEvent(si, in_free[s], 0));
        RT_CUDA_TRY(cudaMemcpyAsync(S.o, in.o + 3 * b, 24 * m, cudaMemcpyHostToDevice, si));
        RT_CUDA_TRY(cudaMemcpyAsync(S.d, in.d + 3 * b, 24 * m, cudaMemcpyHostToDevice, si));
        if (in.tmin) RT_CUDA_TRY(cudaMemcpyAsync(S.tmin, in.tmin + b, 8 * m, cudaMemcpyHostToDevice, si));
        if (in.tmax) RT_CUDA_TRY(cudaMemcpyAsync(S.tmax, in.tmax + b, 8 * m, cudaMemcpyHostToDevice, si));
        RT_CUDA_TRY(cudaEventRecord(in_ready[s], si));
        RT_CUDA_TRY(cudaStreamWaitEvent(sc, in_ready[s], 0));
        if (k >= 2) RT_CUDA_TRY(cudaStreamWaitEvent(sc, out_free[s], 0));
        rc = rt_pack_rays_io(c, m, S, in.tmin != nullptr, in.tmax != nullptr, in.tmin_s, in.tmax_s);
        if (rc) return rc;
        rc = kernels(S, m);
        if (rc) return rc;
        // the slot's float64 inputs are read up to here (the closest-hit expand refines
        // (t, u, v) from them), so the next upload into this slot waits for the kernels
        RT_CUDA_TRY(cudaEventRecord(in_free[s], sc));
        RT_CUDA_TRY(cudaEventRecord(c->io_ev[7 + s], sc));
        RT_CUDA_TRY(cudaStreamWaitEvent(so, c->io_ev[7 + s], 0));
        rc = download(S, b, m, so);
        if (rc) return rc;
        RT_CUDA_TRY(cudaEventRecord(out_free[s], so));
    }
    RT_CUDA_TRY(cudaStreamSynchronize(so));
    RT_CUDA_TRY(cudaStreamSynchronize(sc));
    RT_CUDA_TRY(cudaStreamSynchronize(si));
    return RT_OK;
}
