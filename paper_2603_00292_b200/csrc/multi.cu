// multi.cu -- the multi-GPU data plane: the only exchange of the path is
// the accumulation buffers going to GPU 0 after the renders, over NCCL on NVLink /
// NVSwitch.  Two splits, both with the scene and its LBVH replicated per GPU:
//
//   samples (path tracing): GPU g renders global samples [g*S/N, (g+1)*S/N) of every
//     pixel (its random numbers are those of a 1-GPU run, sampling.py:67-73), then ONE
//     ncclReduce(sum, fp32) of the (H*W, 4) buffers into GPU 0;
//   tiles (primary rays): GPU g renders the interleaved 4-row tile bands r % N == g, packs
//     just those rows into a compact buffer and sends it to GPU 0, which unpacks them into
//     its frame: GPU 0 receives (N-1)/N of one frame instead of reducing N full frames.
//
// One implementation serves both launch modes:
//   * one process per GPU (torch.distributed for the rendezvous only): rt_comm_create per
//     rank from a unique id, rt_comm_gather_bands / rt_comm_reduce_accum per frame;
//   * one process driving N GPUs (rt_multi_render, the CLI's --gpus N): communicators from
//     ncclCommInitAll, every device's share enqueued first, then the same exchange.
// NCCL is loaded with dlopen at the first use: the process shares the libnccl.so.2 already
// loaded (PyTorch's); librt_b200 has no link-time NCCL dependency.
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "rt_common.cuh"

namespace {

typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
struct ncclUniqueId {
    char internal[RT_COMM_ID_BYTES];
};
constexpr int NCCL_SUM = 0, NCCL_FLOAT32 = 7;

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*reduce)(const void*, void*, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    return n;
}

std::mutex& nccl_lock() {
    static std::mutex m;
    return m;
}

int load_nccl() {
    Nccl& n = nccl();
    if (n.h) return RT_OK;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        rt_set_error("cannot load NCCL (libnccl.so.2): %s", dlerror());
        return RT_ECUDA;
    }
#define SYM(f, name) n.f = (decltype(n.f))dlsym(h, name)
    SYM(getUniqueId, "ncclGetUniqueId");
    SYM(commInitRank, "ncclCommInitRank");
    SYM(commInitAll, "ncclCommInitAll");
    SYM(commDestroy, "ncclCommDestroy");
    SYM(reduce, "ncclReduce");
    SYM(send, "ncclSend");
    SYM(recv, "ncclRecv");
    SYM(groupStart, "ncclGroupStart");
    SYM(groupEnd, "ncclGroupEnd");
    SYM(errorString, "ncclGetErrorString");
#undef SYM
    if (!n.getUniqueId || !n.commInitRank || !n.commInitAll || !n.commDestroy || !n.reduce || !n.send || !n.recv ||
        !n.groupStart || !n.groupEnd || !n.errorString) {
        rt_set_error("NCCL library lacks a required symbol");
        return RT_ECUDA;
    }
    n.h = h;
    return RT_OK;
}

#define RT_NCCL_TRY(expr)                                                                     \
    do {                                                                                      \
        ncclResult_t _r = (expr);                                                             \
        if (_r != 0) {                                                                        \
            rt_set_error("%s failed: %s", #expr, nccl().errorString(_r));                     \
            return RT_ENCCL;                                                                  \
        }                                                                                     \
    } while (0)

// ---- interleaved 4-row tile bands (render.cu unit_pixel with band_stride / offset) ----
// rows of rank g of G: bands r = g, g + G, ... of rows [4r, min(4r + 4, H))
int64_t band_rows_of(int32_t height, int g, int G) {
    int64_t rows = 0;
    const int64_t trows = (height + 3) / 4;
    for (int64_t r = g; r < trows; r += G) rows += std::min<int64_t>(4, height - 4 * r);
    return rows;
}

// compact row c of rank g <-> frame row 4 * (g + (c / 4) * G) + c % 4 (only the frame's
// last band can be short, and it is the last band of its rank, so the mapping holds)
__global__ void bands_pack_kernel(const float4* __restrict__ accum, float4* __restrict__ compact, int32_t width,
                                  int64_t rows, int g, int G) {
    const int64_t total = rows * width;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = p / width, x = p - c * width;
        const int64_t row = 4 * (g + (c >> 2) * (int64_t)G) + (c & 3);
        compact[p] = accum[row * width + x];
    }
}

__global__ void bands_unpack_kernel(const float4* __restrict__ compact, float4* __restrict__ accum, int32_t width,
                                    int64_t rows, int g, int G) {
    const int64_t total = rows * width;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = p / width, x = p - c * width;
        const int64_t row = 4 * (g + (c >> 2) * (int64_t)G) + (c & 3);
        accum[row * width + x] = compact[p];
    }
}

unsigned copy_grid(rt_ctx* c, int64_t n) {
    int64_t g = (n + 255) / 256;
    const int64_t cap = (int64_t)c->num_sms * 8;
    return (unsigned)(g < cap ? (g > 0 ? g : 1) : cap);
}

// per-context staging for the band exchange (grown on demand, pool memory)
struct Stage {
    void* p = nullptr;
    size_t bytes = 0;
};
std::map<rt_ctx*, Stage>& stages() {
    static std::map<rt_ctx*, Stage> m;
    return m;
}
std::mutex& stage_lock() {
    static std::mutex m;
    return m;
}
int stage_get(rt_ctx* c, size_t bytes, void** out) {
    std::lock_guard<std::mutex> lk(stage_lock());
    Stage& s = stages()[c];
    if (s.bytes < bytes) {
        if (s.p) {
            RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
            rt_free(s.p, c->stream);
        }
        s.p = nullptr;
        s.bytes = 0;
        RT_CUDA_TRY(rt_alloc(&s.p, bytes, c->stream));
        s.bytes = bytes;
    }
    *out = s.p;
    return RT_OK;
}

// One participant of a band gather: its rank, communicator, context and frame.
struct Part {
    int rank;
    ncclComm_t comm;
    rt_ctx* ctx;
    float* accum;
};

// The band gather for the participants driven by this call (all G ranks in one process,
// or one rank per process): pack on every non-root rank, one NCCL group of sends to rank
// 0 and receives on rank 0, unpack on rank 0.  Everything on the contexts' streams.
int gather_bands(const std::vector<Part>& parts, int G, int32_t width, int32_t height) {
    std::vector<int64_t> rows(G), off(G + 1, 0);
    for (int g = 0; g < G; ++g) {
        rows[g] = band_rows_of(height, g, G);
        off[g + 1] = off[g] + (g == 0 ? 0 : rows[g]);         // root's staging: ranks 1..G-1
    }
    std::vector<void*> buf(parts.size(), nullptr);
    for (size_t k = 0; k < parts.size(); ++k) {
        const Part& P = parts[k];
        RT_CUDA_TRY(cudaSetDevice(P.ctx->device));
        const size_t bytes = (size_t)(P.rank == 0 ? off[G] : rows[P.rank]) * width * sizeof(float4);
        if (bytes == 0) continue;
        int rc = stage_get(P.ctx, bytes, &buf[k]);
        if (rc) return rc;
        if (P.rank != 0) {
            bands_pack_kernel<<<copy_grid(P.ctx, rows[P.rank] * width), 256, 0, P.ctx->stream>>>(
                reinterpret_cast<const float4*>(P.accum), reinterpret_cast<float4*>(buf[k]), width, rows[P.rank],
                P.rank, G);
            RT_CUDA_TRY(cudaGetLastError());
        }
    }
    RT_NCCL_TRY(nccl().groupStart());
    for (size_t k = 0; k < parts.size(); ++k) {
        const Part& P = parts[k];
        if (P.rank != 0) {
            if (rows[P.rank])
                RT_NCCL_TRY(nccl().send(buf[k], (size_t)rows[P.rank] * width * 4, NCCL_FLOAT32, 0, P.comm,
                                        P.ctx->stream));
        } else {
            for (int g = 1; g < G; ++g)
                if (rows[g])
                    RT_NCCL_TRY(nccl().recv(reinterpret_cast<float4*>(buf[k]) + off[g] * width,
                                            (size_t)rows[g] * width * 4, NCCL_FLOAT32, g, P.comm, P.ctx->stream));
        }
    }
    RT_NCCL_TRY(nccl().groupEnd());
    for (size_t k = 0; k < parts.size(); ++k) {
        const Part& P = parts[k];
        if (P.rank != 0) continue;
        RT_CUDA_TRY(cudaSetDevice(P.ctx->device));
        for (int g = 1; g < G; ++g)
            if (rows[g])
                bands_unpack_kernel<<<copy_grid(P.ctx, rows[g] * width), 256, 0, P.ctx->stream>>>(
                    reinterpret_cast<const float4*>(buf[k]) + off[g] * width, reinterpret_cast<float4*>(P.accum),
                    width, rows[g], g, G);
        RT_CUDA_TRY(cudaGetLastError());
    }
    return RT_OK;
}

// communicators per device list for the single-process path, created once
// (ncclCommInitAll is expensive)
std::map<std::vector<int>, std::vector<ncclComm_t>>& comm_cache() {
    static std::map<std::vector<int>, std::vector<ncclComm_t>> m;
    return m;
}

}  // namespace

struct rt_comm {
    int nranks, rank, device;
    ncclComm_t comm;
};

extern "C" {

int rt_comm_unique_id(uint8_t* id) {
    RT_CHECK_ARG(id, "NULL id buffer");
    std::lock_guard<std::mutex> lk(nccl_lock());
    int rc = load_nccl();
    if (rc) return rc;
    ncclUniqueId u;
    RT_NCCL_TRY(nccl().getUniqueId(&u));
    memcpy(id, u.internal, RT_COMM_ID_BYTES);
    return RT_OK;
}

int rt_comm_create(rt_ctx* c, int32_t nranks, int32_t rank, const uint8_t* id, rt_comm** out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(id && out && nranks >= 1 && rank >= 0 && rank < nranks, "bad communicator arguments");
    {
        std::lock_guard<std::mutex> lk(nccl_lock());
        int rc = load_nccl();
        if (rc) return rc;
    }
    RT_CUDA_TRY(cudaSetDevice(c->device));
    ncclUniqueId u;
    memcpy(u.internal, id, RT_COMM_ID_BYTES);
    ncclComm_t comm = nullptr;
    RT_NCCL_TRY(nccl().commInitRank(&comm, nranks, u, rank));
    rt_comm* m = new rt_comm();
    m->nranks = nranks;
    m->rank = rank;
    m->device = c->device;
    m->comm = comm;
    *out = m;
    return RT_OK;
}

void rt_comm_destroy(rt_comm* m) {
    if (!m) return;
    if (m->comm && nccl().commDestroy) nccl().commDestroy(m->comm);
    delete m;
}

int rt_comm_reduce_accum(rt_comm* m, rt_ctx* c, float* accum, int64_t npix) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(m && accum && npix >= 0, "NULL argument");
    RT_CHECK_ARG(m->device == c->device, "communicator and context live on different devices");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_NCCL_TRY(nccl().reduce(accum, accum, (size_t)npix * 4, NCCL_FLOAT32, NCCL_SUM, 0, m->comm, c->stream));
    return RT_OK;
}

int rt_comm_gather_bands(rt_comm* m, rt_ctx* c, float* accum, int32_t width, int32_t height) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(m && accum && width >= 1 && height >= 1, "bad gather arguments");
    RT_CHECK_ARG(m->device == c->device, "communicator and context live on different devices");
    if (m->nranks == 1) return RT_OK;
    return gather_bands({Part{m->rank, m->comm, c, accum}}, m->nranks, width, height);
}

// test hook: the band gather's pack / unpack index math on one device (no NCCL):
// compact = rank g's rows of accum (pack) or accum rows from compact (unpack)
int rt_bands_copy(rt_ctx* c, float* accum, float* compact, int32_t width, int32_t height, int32_t g, int32_t G,
                  int32_t unpack, int64_t* rows_out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(accum && compact && width >= 1 && height >= 1 && G >= 1 && g >= 0 && g < G, "bad band arguments");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    const int64_t rows = band_rows_of(height, g, G);
    if (rows_out) *rows_out = rows;
    if (rows == 0) return RT_OK;
    if (unpack)
        bands_unpack_kernel<<<copy_grid(c, rows * width), 256, 0, c->stream>>>(
            reinterpret_cast<const float4*>(compact), reinterpret_cast<float4*>(accum), width, rows, g, G);
    else
        bands_pack_kernel<<<copy_grid(c, rows * width), 256, 0, c->stream>>>(
            reinterpret_cast<const float4*>(accum), reinterpret_cast<float4*>(compact), width, rows, g, G);
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

int rt_multi_render(int32_t n_gpus, rt_ctx* const* ctxs, rt_scene* const* scenes, const rt_render_params* p,
                    float* const* accums, int32_t split, uint64_t* rays_out) {
    RT_CHECK_ARG(n_gpus >= 1 && ctxs && scenes && p && accums, "NULL argument");
    RT_CHECK_ARG(split == RT_SPLIT_SAMPLES || split == RT_SPLIT_TILES, "split must be samples or tiles");
    RT_CHECK_ARG(p->s1 > p->s0 && p->s0 >= 0, "width, height, and spp must all be >= 1");
    std::vector<int> devs(n_gpus);
    for (int g = 0; g < n_gpus; ++g) {
        RT_CHECK_ARG(ctxs[g] && scenes[g] && accums[g], "NULL context, scene or accumulation buffer");
        if (!scenes[g]->built) { rt_set_error("BVH not built on device %d", ctxs[g]->device); return RT_ESTATE; }
        devs[g] = ctxs[g]->device;
        for (int k = 0; k < g; ++k)
            RT_CHECK_ARG(devs[k] != devs[g], "every replica must live on a distinct device");
    }
    // hold every context's lock (in address order: no lock-order inversion between callers)
    std::vector<rt_ctx*> order(ctxs, ctxs + n_gpus);
    std::sort(order.begin(), order.end());
    std::vector<std::unique_lock<std::recursive_mutex>> locks;
    for (rt_ctx* c : order) locks.emplace_back(*c->mu);
    const int64_t npix = (int64_t)p->width * p->height;
    RT_CHECK_ARG(p->pix_lo == 0 && (p->pix_hi == 0 || p->pix_hi == npix), "multi-GPU renders whole frames");
    // 1. every device's share, enqueued without waiting (renders run concurrently)
    const int64_t spp = p->s1 - p->s0;
    std::vector<char> rendered(n_gpus, 0);
    for (int g = 0; g < n_gpus; ++g) {
        rt_render_params q = *p;
        if (split == RT_SPLIT_SAMPLES) {
            q.s0 = (int32_t)(p->s0 + g * spp / n_gpus);
            q.s1 = (int32_t)(p->s0 + (g + 1) * spp / n_gpus);
            if (q.s1 <= q.s0) continue;
        } else {
            q.band_stride = n_gpus;
            q.band_offset = g;
        }
        RT_CUDA_TRY(cudaSetDevice(devs[g]));
        int rc = rt_render_impl(ctxs[g], scenes[g], &q, accums[g], nullptr);
        if (rc) return rc;
        rendered[g] = 1;
    }
    // 2. the exchange: reduce (samples) or band gather (tiles) into device 0
    //    (RT_MULTI_FORCE_NCCL=1 runs the reduce for one device too: the NCCL plumbing is
    //    then testable on a 1-GPU box)
    static const bool force = getenv("RT_MULTI_FORCE_NCCL") != nullptr;
    if (n_gpus > 1 || force) {
        std::lock_guard<std::mutex> lk(nccl_lock());
        int rc = load_nccl();
        if (rc) return rc;
        auto& cc = comm_cache();
        auto it = cc.find(devs);
        if (it == cc.end()) {
            std::vector<ncclComm_t> comms(n_gpus);
            RT_NCCL_TRY(nccl().commInitAll(comms.data(), n_gpus, devs.data()));
            it = cc.emplace(devs, comms).first;
        }
        if (split == RT_SPLIT_TILES && n_gpus > 1) {
            std::vector<Part> parts;
            for (int g = 0; g < n_gpus; ++g) parts.push_back(Part{g, it->second[g], ctxs[g], accums[g]});
            rc = gather_bands(parts, n_gpus, p->width, p->height);
            if (rc) return rc;
        } else {
            RT_NCCL_TRY(nccl().groupStart());
            for (int g = 0; g < n_gpus; ++g)
                RT_NCCL_TRY(nccl().reduce(accums[g], accums[0], (size_t)npix * 4, NCCL_FLOAT32, NCCL_SUM, 0,
                                          it->second[g], ctxs[g]->stream));
            RT_NCCL_TRY(nccl().groupEnd());
        }
    }
    // 3. wait, sum the closest-hit query counts, surface device errors
    uint64_t total = 0;
    for (int g = 0; g < n_gpus; ++g) {
        RT_CUDA_TRY(cudaSetDevice(devs[g]));
        if (!rendered[g]) {                      // more devices than samples: nothing ran here
            RT_CUDA_TRY(cudaStreamSynchronize(ctxs[g]->stream));
            continue;
        }
        unsigned long long r = 0;
        RT_CUDA_TRY(cudaMemcpyAsync(&r, ctxs[g]->d_counter + 32, sizeof r, cudaMemcpyDeviceToHost, ctxs[g]->stream));
        RT_CUDA_TRY(cudaStreamSynchronize(ctxs[g]->stream));
        int rc = rt_check_device_error(ctxs[g]);
        if (rc) return rc;
        total += r;
    }
    if (rays_out) *rays_out = total;
    return RT_OK;
}

}  // extern "C"
