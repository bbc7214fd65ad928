// multi.cu -- single-process multi-GPU render (rt_multi_render): the work split of
// SURVEY 8(e) on N devices of one node plus ONE NCCL reduce of the fp32 accumulation
// buffers into device 0 (NVLink / NVSwitch; NVLS-eligible).
//
//   samples (path tracing): device g renders global samples [g*S/N, (g+1)*S/N) of every
//     pixel, so its random numbers are those of a 1-GPU run (sampling.py:67-73);
//   tiles (primary rays): device g renders the interleaved 4-row tile bands r % N == g
//     (untouched pixels stay 0, so the same sum assembles the frame).
//
// All renders are enqueued first (one context stream per device, nothing waits), then
// the grouped ncclReduce, then the ray counters are read.  NCCL is loaded with dlopen
// at the first call: the process shares whatever libnccl.so.2 is already loaded
// (PyTorch's), and librt_b200 itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <vector>

#include "rt_common.cuh"

namespace {

typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
constexpr int NCCL_SUM = 0, NCCL_FLOAT32 = 7;

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*reduce)(const void*, void*, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
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
    n.commInitAll = (decltype(n.commInitAll))dlsym(h, "ncclCommInitAll");
    n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
    n.reduce = (decltype(n.reduce))dlsym(h, "ncclReduce");
    n.groupStart = (decltype(n.groupStart))dlsym(h, "ncclGroupStart");
    n.groupEnd = (decltype(n.groupEnd))dlsym(h, "ncclGroupEnd");
    n.errorString = (decltype(n.errorString))dlsym(h, "ncclGetErrorString");
    if (!n.commInitAll || !n.commDestroy || !n.reduce || !n.groupStart || !n.groupEnd || !n.errorString) {
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

// communicators per device list, created once (ncclCommInitAll is expensive)
std::map<std::vector<int>, std::vector<ncclComm_t>>& comm_cache() {
    static std::map<std::vector<int>, std::vector<ncclComm_t>> m;
    return m;
}

}  // namespace

extern "C" {

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
    // 2. one reduce(sum) of the (H*W, 4) fp32 buffers into device 0 (RT_MULTI_FORCE_NCCL=1
    //    runs it for one device too: the NCCL plumbing is then testable on a 1-GPU box)
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
        RT_NCCL_TRY(nccl().groupStart());
        for (int g = 0; g < n_gpus; ++g)
            RT_NCCL_TRY(nccl().reduce(accums[g], accums[0], (size_t)npix * 4, NCCL_FLOAT32, NCCL_SUM, 0,
                                      it->second[g], ctxs[g]->stream));
        RT_NCCL_TRY(nccl().groupEnd());
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
