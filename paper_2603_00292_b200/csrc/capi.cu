// capi.cu -- the extern "C" boundary of librt_b200.so (declared in include/rt_b200.h).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "hostio.cuh"
#include "rt_common.cuh"

static thread_local char g_err[1024] = "";

void rt_set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

size_t rt_sort_scratch_words(int64_t n);
void rt_render_release(rt_scene* s);



// Host -> device copy of a caller's array.  Pinned (page-locked) sources go as one async
// DMA.  Large pageable ones (numpy arrays: compile_scene's float64 vertices / int64 faces)
// are staged: host threads copy 16-MB chunks into two pinned buffers of the context while
// the copy engine moves the previous chunk (the driver's own pageable path stages with one
// thread: ~11 GB/s measured for the 10M soup's 960 MB).  Returns after the source may be
// reused (the last chunk is in a pinned buffer or on the device).
int rt_h2d(rt_ctx* c, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return RT_OK;
    cudaPointerAttributes a;
    const bool pinned = cudaPointerGetAttributes(&a, src) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();                       // (unregistered pointers may set a sticky-free error)
    constexpr size_t CHUNK = 16u << 20;
    if (pinned || bytes <= 2 * CHUNK) {
        RT_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
        return RT_OK;
    }
    if (!c->h_stage) {
        RT_CUDA_TRY(cudaHostAlloc(&c->h_stage, 2 * CHUNK, cudaHostAllocDefault));
        c->h_stage_bytes = 2 * CHUNK;
        RT_CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev[0], cudaEventDisableTiming));
        RT_CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev[1], cudaEventDisableTiming));
    }
    const unsigned hw = std::thread::hardware_concurrency();
    const int nt = (int)std::max(1u, std::min(8u, hw / 2));
    const char* s8 = static_cast<const char*>(src);
    char* d8 = static_cast<char*>(dst);
    for (size_t off = 0, k = 0; off < bytes; off += CHUNK, ++k) {
        const size_t len = std::min(CHUNK, bytes - off);
        char* buf = static_cast<char*>(c->h_stage) + (k & 1) * CHUNK;
        if (k >= 2) RT_CUDA_TRY(cudaEventSynchronize(c->stage_ev[k & 1]));   // buffer free again
        const size_t per = (len + nt - 1) / nt;
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) {
            const size_t a0 = std::min(len, t * per), a1 = std::min(len, (t + 1) * per);
            if (a1 > a0) th.emplace_back([=] { memcpy(buf + a0, s8 + off + a0, a1 - a0); });
        }
        memcpy(buf, s8 + off, std::min(len, per));
        for (auto& x : th) x.join();
        RT_CUDA_TRY(cudaMemcpyAsync(d8 + off, buf, len, cudaMemcpyHostToDevice, c->stream));
        RT_CUDA_TRY(cudaEventRecord(c->stage_ev[k & 1], c->stream));
    }
    // the staging buffers are reused by the next call: their last copies must be done
    RT_CUDA_TRY(cudaEventSynchronize(c->stage_ev[0]));
    RT_CUDA_TRY(cudaEventSynchronize(c->stage_ev[1]));
    return RT_OK;
}

int rt_check_device_error(rt_ctx* ctx) {
    int e = 0;
    RT_CUDA_TRY(cudaMemcpyAsync(&e, ctx->d_error, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
    RT_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (e == 0) return RT_OK;
    int z = 0;
    cudaMemcpy(ctx->d_error, &z, sizeof z, cudaMemcpyHostToDevice);
    if (e == RT_EDEPTH) {
        rt_set_error("BVH height exceeds the %d-entry traversal stack", RT_STACK - 1);
        return RT_EDEPTH;
    }
    if (e == RT_EUNSUPPORTED) {
        rt_set_error("a ray reached a custom primitive with no intersection function registered");
        return RT_EUNSUPPORTED;
    }
    rt_set_error("device error %d", e);
    return RT_ECUDA;
}

extern "C" {

const char* rt_last_error(void) { return g_err; }
const char* rt_version(void) { return "librt_b200 0.1 (sm_100a)"; }

int rt_device_count(int* n) {
    RT_CUDA_TRY(cudaGetDeviceCount(n));
    return RT_OK;
}

int rt_ctx_create(int device, rt_ctx** out) {
    RT_CHECK_ARG(out != nullptr, "out is NULL");
    int n = 0;
    RT_CUDA_TRY(cudaGetDeviceCount(&n));
    RT_CHECK_ARG(device >= 0 && device < n, "device index out of range");
    RT_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    RT_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
        rt_set_error("librt_b200 targets sm_100a (B200); device %d is sm_%d%d", device, prop.major, prop.minor);
        return RT_ECUDA;
    }
    rt_ctx* c = new rt_ctx();
    memset(c, 0, sizeof *c);
    c->mu = new std::recursive_mutex();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    RT_CUDA_TRY(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    RT_CUDA_TRY(cudaEventCreate(&c->ev0));
    RT_CUDA_TRY(cudaEventCreate(&c->ev1));
    {
        // keep freed pool blocks cached (scene storage is stream-ordered pool memory)
        cudaMemPool_t pool;
        RT_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        RT_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    RT_CUDA_TRY(cudaMalloc(&c->d_counter, 64 * sizeof(unsigned int)));
    RT_CUDA_TRY(cudaMalloc(&c->d_error, sizeof(int)));
    RT_CUDA_TRY(cudaMemset(c->d_error, 0, sizeof(int)));
    *out = c;
    return RT_OK;
}

void rt_ctx_destroy(rt_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->h_stage) {
        cudaFreeHost(c->h_stage);
        cudaEventDestroy(c->stage_ev[0]);
        cudaEventDestroy(c->stage_ev[1]);
    }
    if (c->d_stage) cudaFree(c->d_stage);
    if (c->d_io) cudaFree(c->d_io);
    if (c->io_in) {
        cudaStreamSynchronize(c->io_in);
        cudaStreamSynchronize(c->io_out);
        cudaStreamDestroy(c->io_in);
        cudaStreamDestroy(c->io_out);
        for (int k = 0; k < 9; ++k) cudaEventDestroy(c->io_ev[k]);
    }
    cudaFree(c->d_counter);
    cudaFree(c->d_error);
    if (c->d_probe) cudaFree(c->d_probe);
    if (c->d_chunk_done) cudaFree(c->d_chunk_done);
    if (c->d_rb) cudaFree(c->d_rb);
    if (c->h_tab) cudaFreeHost(c->h_tab);
    if (c->tab_ev) cudaEventDestroy(c->tab_ev);
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    cudaStreamDestroy(c->own_stream);
    delete c->mu;
    delete c;
}

int rt_ctx_counters(rt_ctx* c, uint32_t* out64) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(out64, "NULL output");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_CUDA_TRY(cudaMemcpyAsync(out64, c->d_counter, 64 * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return RT_OK;
}

int rt_ctx_set_stream(rt_ctx* c, void* stream) {
    RT_CHECK_ARG(c, "ctx is NULL");
    c->stream = (cudaStream_t)stream;   // used verbatim: NULL is the legacy default stream
    return RT_OK;
}

int rt_ctx_sync(rt_ctx* c) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c, "ctx is NULL");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return rt_check_device_error(c);
}

// device allocations of a scene of n primitives and n_mat materials (contents unset)
int rt_scene_alloc(rt_ctx* c, int64_t n, int32_t n_mat, rt_scene** out) { return rt_scene_alloc_ex(c, n, n_mat, out, 1); }

// sync = 0: the caller synchronises the context stream before the scene is used from
// another stream (rt_scene_compile behind pending mesh uploads: rt_mesh_upload_finish)
int rt_scene_alloc_ex(rt_ctx* c, int64_t n, int32_t n_mat, rt_scene** out, int sync) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && out, "ctx/out is NULL");
    RT_CHECK_ARG(n >= 1, "cannot build over zero primitives");
    RT_CHECK_ARG(n < (1ll << 30), "at most 2^30 - 1 triangles per scene");
    RT_CHECK_ARG(n_mat >= 1, "materials missing");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_scene* s = new rt_scene();
    memset(s, 0, sizeof *s);
    s->n = n;
    s->n_mat = n_mat;
    s->device = c->device;
    s->stream = c->stream;
    const int64_t ni = n > 1 ? n - 1 : 1;
#define ALLOC(ptr, bytes)                                                       \
    do {                                                                        \
        cudaError_t _e = rt_alloc((void**)&(ptr), (bytes), c->stream, false);   \
        if (_e != cudaSuccess) {                                                \
            rt_set_error("cudaMalloc(%zu) failed: %s", (size_t)(bytes), cudaGetErrorString(_e)); \
            rt_scene_destroy(s);                                                \
            return RT_ENOMEM;                                                   \
        }                                                                       \
    } while (0)
    ALLOC(s->tris, sizeof(float) * 9 * n + 64);     // + the last rows' 64-B gather window (lbvh.cu)
    ALLOC(s->tri_attr, sizeof(float4) * n);
    ALLOC(s->tri_inst, sizeof(int32_t) * n);
    ALLOC(s->tri_prim, sizeof(int32_t) * n);
    ALLOC(s->tri_mask, sizeof(uint32_t) * n);
    ALLOC(s->mat_color, sizeof(float4) * n_mat);
    ALLOC(s->mat_emissive, sizeof(float4) * n_mat);
    ALLOC(s->nodes, sizeof(float4) * 4);          // root record (the binary view is derived on download)
    ALLOC(s->tri_sorted, sizeof(float4) * 3 * n);
    ALLOC(s->bvh4, sizeof(float4) * 8 * ni);
    ALLOC(s->keys_a, sizeof(uint64_t) * n);
    ALLOC(s->keys_b, sizeof(uint64_t) * n);
    ALLOC(s->vals_a, sizeof(uint32_t) * n);
    ALLOC(s->vals_b, sizeof(uint32_t) * n);
    ALLOC(s->child, sizeof(int2) * ni);
    ALLOC(s->flags, sizeof(unsigned int) * ni);
    ALLOC(s->cbounds, sizeof(float) * 16);
    s->sort_scratch_words = rt_sort_scratch_words(n);
    ALLOC(s->sort_scratch, sizeof(unsigned int) * s->sort_scratch_words);
    ALLOC(s->leaf_box, sizeof(float4) * 4 * n);   // per split slot: (lo, h), hi for both sides
    ALLOC(s->emit_items, 48 * (2 * n + 512));      // EmitNode segments of EMIT_T per emit block
    ALLOC(s->seg_count, sizeof(unsigned int) * (n / 64 + 2));   // one count per emit block (EMIT_T >= 64)
#undef ALLOC
    {
        // the sort scratch starts zeroed; after that every build's last kernel zeroes it again
        // for the next build (lbvh.cu), so no build pays a memset up front
        cudaError_t _e = cudaMemsetAsync(s->sort_scratch, 0, sizeof(unsigned int) * s->sort_scratch_words, c->stream);
        if (_e != cudaSuccess) {
            rt_set_error("cudaMemsetAsync failed: %s", cudaGetErrorString(_e));
            rt_scene_destroy(s);
            return RT_ECUDA;
        }
    }
    if (reinterpret_cast<uintptr_t>(s->tris) & 31) {     // the build's 256-bit row gathers
        rt_set_error("triangle rows are not 32-B aligned");
        rt_scene_destroy(s);
        return RT_ECUDA;
    }
    if (sync) {
        cudaError_t _e = cudaStreamSynchronize(c->stream);   // the blocks are usable from any stream now
        if (_e != cudaSuccess) {
            rt_set_error("allocation failed: %s", cudaGetErrorString(_e));
            rt_scene_destroy(s);
            return RT_ENOMEM;
        }
    }
    *out = s;
    return RT_OK;
}

int rt_scene_set_materials(rt_ctx* c, rt_scene* s, const float* mat_color, const float* mat_emissive) {
    RT_CTX_LOCK(c);
    RT_CUDA_TRY(cudaSetDevice(c->device));      // the scene's buffers live on the context's device
    std::vector<float4> mc(s->n_mat), me(s->n_mat);
    for (int k = 0; k < s->n_mat; ++k) {
        mc[k] = make_float4(mat_color[3 * k], mat_color[3 * k + 1], mat_color[3 * k + 2], 0.f);
        me[k] = make_float4(mat_emissive[3 * k], mat_emissive[3 * k + 1], mat_emissive[3 * k + 2], 0.f);
    }
    // (pageable sources are staged before an async H2D returns: the vectors may go)
    RT_CUDA_TRY(cudaMemcpyAsync(s->mat_color, mc.data(), sizeof(float4) * s->n_mat, cudaMemcpyHostToDevice, c->stream));
    RT_CUDA_TRY(
        cudaMemcpyAsync(s->mat_emissive, me.data(), sizeof(float4) * s->n_mat, cudaMemcpyHostToDevice, c->stream));
    return RT_OK;
}

int rt_scene_create(rt_ctx* c, int64_t n, const float* tris, const float* normals, const int32_t* tri_inst,
                    const int32_t* tri_prim, const uint32_t* tri_mask, const int32_t* tri_material,
                    const float* mat_color, const float* mat_emissive, int32_t n_mat, rt_scene** out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && out, "ctx/out is NULL");
    RT_CHECK_ARG(n >= 1, "cannot build over zero primitives");
    RT_CHECK_ARG(tris && normals && tri_inst && tri_prim && tri_mask && tri_material, "NULL triangle array");
    RT_CHECK_ARG(n_mat >= 1 && mat_color && mat_emissive, "materials missing");
    for (int64_t i = 0; i < n; ++i)
        if (tri_material[i] < 0 || tri_material[i] >= n_mat) {
            rt_set_error("triangle %lld references material %d of %d", (long long)i, tri_material[i], n_mat);
            return RT_EINVAL;
        }
    rt_scene* s = nullptr;
    int rc = rt_scene_alloc(c, n, n_mat, &s);
    if (rc) return rc;
    std::vector<float4> attr(n);
    for (int64_t i = 0; i < n; ++i) {
        float4 a;
        a.x = normals[3 * i]; a.y = normals[3 * i + 1]; a.z = normals[3 * i + 2];
        int m = tri_material[i];
        memcpy(&a.w, &m, 4);
        attr[i] = a;
    }
    cudaStream_t st = c->stream;
    auto fail = [&](cudaError_t e) {
        rt_set_error("upload failed: %s", cudaGetErrorString(e));
        rt_scene_destroy(s);
        return RT_ECUDA;
    };
    cudaError_t e;
    if ((e = cudaMemcpyAsync(s->tris, tris, sizeof(float) * 9 * n, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(s->tri_attr, attr.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(s->tri_inst, tri_inst, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(s->tri_prim, tri_prim, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(s->tri_mask, tri_mask, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st)) ||
        (e = cudaStreamSynchronize(st)))   // host vectors go out of scope
        return fail(e);
    rc = rt_scene_set_materials(c, s, mat_color, mat_emissive);
    if (rc) { rt_scene_destroy(s); return rc; }
    s->mask_uniform = 1;
    s->mask_value = tri_mask[0];
    for (int64_t i = 1; i < n && s->mask_uniform; ++i) s->mask_uniform = tri_mask[i] == tri_mask[0];
    *out = s;
    return RT_OK;
}

int rt_scene_set_vertices(rt_ctx* c, rt_scene* s, const float* tris) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && tris, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_CUDA_TRY(cudaMemcpyAsync(s->tris, tris, sizeof(float) * 9 * s->n, cudaMemcpyHostToDevice, c->stream));
    s->built = 0;
    return RT_OK;
}

// A render replica of a built scene on another context's device (multi-GPU render_frame):
// the resident geometry, shading tables and the built LBVH are copied device to device
// (cudaMemcpyPeer; staged through the host when the devices have no peer access), the
// build scratch is fresh.  The host-query extras (float64 normals / local rows) are not
// copied: a replica renders.
int rt_scene_clone(rt_ctx* src, rt_scene* s, rt_ctx* dst, rt_scene** out) {
    RT_CHECK_ARG(src && s && dst && out, "NULL argument");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    std::unique_lock<std::recursive_mutex> l1(*src->mu, std::defer_lock), l2(*dst->mu, std::defer_lock);
    if (src == dst) l1.lock();
    else if (src < dst) { l1.lock(); l2.lock(); }
    else { l2.lock(); l1.lock(); }
    RT_CUDA_TRY(cudaSetDevice(src->device));
    RT_CUDA_TRY(cudaStreamSynchronize(src->stream));
    rt_scene* d = nullptr;
    int rc = rt_scene_alloc(dst, s->n, s->n_mat, &d);
    if (rc) return rc;
    const int64_t n = s->n, ni = n > 1 ? n - 1 : 1;
    cudaStream_t st = dst->stream;
    auto cp = [&](void* to, const void* from, size_t bytes) -> cudaError_t {
        return cudaMemcpyPeerAsync(to, dst->device, from, src->device, bytes, st);
    };
    cudaError_t e = cudaSuccess;
    if (!e) e = cp(d->tris, s->tris, sizeof(float) * 9 * n);
    if (!e) e = cp(d->tri_attr, s->tri_attr, sizeof(float4) * n);
    if (!e) e = cp(d->tri_inst, s->tri_inst, sizeof(int32_t) * n);
    if (!e) e = cp(d->tri_prim, s->tri_prim, sizeof(int32_t) * n);
    if (!e) e = cp(d->tri_mask, s->tri_mask, sizeof(uint32_t) * n);
    if (!e) e = cp(d->mat_color, s->mat_color, sizeof(float4) * s->n_mat);
    if (!e) e = cp(d->mat_emissive, s->mat_emissive, sizeof(float4) * s->n_mat);
    if (!e) e = cp(d->nodes, s->nodes, sizeof(float4) * 4);
    if (!e) e = cp(d->tri_sorted, s->tri_sorted, sizeof(float4) * 3 * n);
    if (!e) e = cp(d->bvh4, s->bvh4, sizeof(float4) * 8 * ni);
    if (!e) e = cp(d->vals_a, s->vals_a, sizeof(uint32_t) * n);
    if (!e) e = cp(d->keys_a, s->keys_a, (s->bits == 63 ? 8 : 4) * (size_t)n);
    if (!e) e = cp(d->cbounds, s->cbounds, sizeof(float) * 16);
    if (!e && s->n_lights) {
        e = rt_alloc((void**)&d->lights, sizeof(float4) * 5 * s->n_lights, st);
        if (!e) e = cp(d->lights, s->lights, sizeof(float4) * 5 * s->n_lights);
        d->n_lights = s->n_lights;
    }
    if (!e && s->n_spheres) {
        e = rt_alloc((void**)&d->spheres, sizeof(double) * 16 * s->n_spheres, st);
        if (!e) e = cp(d->spheres, s->spheres, sizeof(double) * 16 * s->n_spheres);
        d->n_spheres = s->n_spheres;
    }
    if (!e) e = cudaStreamSynchronize(st);
    if (e) {
        rt_scene_destroy(d);
        rt_set_error("rt_scene_clone: %s", cudaGetErrorString(e));
        return RT_ECUDA;
    }
    d->built = s->built;
    d->bits = s->bits;
    d->mask_uniform = s->mask_uniform;
    d->mask_value = s->mask_value;
    d->custom = s->custom;
    d->geom_type = s->geom_type;
    d->data_offset = s->data_offset;
    *out = d;
    return RT_OK;
}

void rt_scene_destroy(rt_scene* s) {
    if (!s) return;
    rt_render_release(s);
    void* ptrs[] = {s->tris, s->tri_attr, s->tri_inst, s->tri_prim, s->tri_mask, s->mat_color, s->mat_emissive,
                    s->nodes, s->tri_sorted, s->bvh4, s->keys_a, s->keys_b, s->vals_a, s->vals_b, s->child,
                    s->flags, s->cbounds, s->sort_scratch, s->leaf_box, s->emit_items, s->seg_count, s->lights,
                    s->spheres,
                    s->lnormal64, s->lrows64, s->wnormal64, s->inst_inv64, s->probe_hint};
    cudaSetDevice(s->device);
    for (void* p : ptrs) rt_free(p, s->stream);
    delete s;
}

int rt_bvh_build(rt_ctx* c, rt_scene* s, int bits, float* build_ms) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "ctx/scene is NULL");
    RT_CHECK_ARG(bits == 30 || bits == 63, "morton_bits must be 30 or 63");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    if (build_ms) RT_CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    int rc = rt_lbvh_build_impl(c, s, bits);
    if (rc) return rc;
    s->built = 1;
    s->bits = bits;
    if (build_ms) {
        RT_CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
        RT_CUDA_TRY(cudaEventSynchronize(c->ev1));
        RT_CUDA_TRY(cudaEventElapsedTime(build_ms, c->ev0, c->ev1));
    }
    return RT_OK;
}

int rt_bvh_build_profiled(rt_ctx* c, rt_scene* s, int bits, float* stage_ms) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && stage_ms, "NULL argument");
    RT_CHECK_ARG(bits == 30 || bits == 63, "morton_bits must be 30 or 63");
    RT_CHECK_ARG(s->n > 1, "profiling needs at least two triangles");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    if (!c->prof[0])
        for (int k = 0; k < 8; ++k) RT_CUDA_TRY(cudaEventCreate(&c->prof[k]));
    c->profiling = 1;
    int rc = rt_lbvh_build_impl(c, s, bits);
    c->profiling = 0;
    if (rc) return rc;
    s->built = 1;
    s->bits = bits;
    RT_CUDA_TRY(cudaEventSynchronize(c->prof[6]));
    for (int k = 0; k < 6; ++k) RT_CUDA_TRY(cudaEventElapsedTime(stage_ms + k, c->prof[k], c->prof[k + 1]));
    return RT_OK;
}

int rt_bvh_info(rt_ctx* c, rt_scene* s, float* root6, int32_t* height, int64_t* n_internal) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "ctx/scene is NULL");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    RT_CUDA_TRY(cudaSetDevice(c->device));
    float4 nd[4];
    RT_CUDA_TRY(cudaMemcpyAsync(nd, s->nodes, sizeof nd, cudaMemcpyDeviceToHost, c->stream));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (root6) {
        root6[0] = std::min(nd[0].x, nd[1].x); root6[3] = std::max(nd[0].y, nd[1].y);
        root6[1] = std::min(nd[0].z, nd[1].z); root6[4] = std::max(nd[0].w, nd[1].w);
        root6[2] = std::min(nd[2].x, nd[2].z); root6[5] = std::max(nd[2].y, nd[2].w);
    }
    if (height) memcpy(height, &nd[3].z, 4);
    if (n_internal) *n_internal = s->n > 1 ? s->n - 1 : 1;
    return RT_OK;
}

int rt_bvh_download(rt_ctx* c, rt_scene* s, uint64_t* sorted_keys, uint32_t* order, int32_t* child,
                    int32_t* parent, float* boxes, int32_t* heights, float* cbounds, float* inv_ext,
                    uint64_t* morton) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "ctx/scene is NULL");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const int64_t n = s->n;
    if (n == 1) {
        if (order) { order[0] = 0; }
        return RT_OK;
    }
    const bool wide = s->bits == 63;
    auto keys_to_u64 = [&](const void* dev, uint64_t* host) -> int {
        if (wide) {
            RT_CUDA_TRY(cudaMemcpy(host, dev, 8 * n, cudaMemcpyDeviceToHost));
        } else {
            std::vector<uint32_t> tmp(n);
            RT_CUDA_TRY(cudaMemcpy(tmp.data(), dev, 4 * n, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < n; ++i) host[i] = tmp[i];
        }
        return RT_OK;
    };
    int rc;
    if (sorted_keys && (rc = keys_to_u64(s->keys_a, sorted_keys))) return rc;
    if (order) RT_CUDA_TRY(cudaMemcpy(order, s->vals_a, 4 * n, cudaMemcpyDeviceToHost));
    if (child || parent || boxes || heights) {
        // the build writes only the BVH4 halves + the root record; the binary view is
        // derived here.  Topology: the half a node W writes into its parent P's entry
        // (entry index = P's split, side = W's side) records W's own split (.w of its first
        // hi vector), so from the root's split (root record) every node's split follows,
        // hence every range [l, r] -> children [l, g], [g + 1, r] and the Karras numbers
        // (a left child is numbered by its right end, a right child by its left end, a
        // leaf k by ~k).  Boxes: node P's child boxes are the half P wrote into its parent
        // Q's entry (the root's are in the root record).  Heights bottom-up; parents by
        // inverting child.
        const int64_t m = n - 1;
        std::vector<float4> b4(8 * m), root(4);
        RT_CUDA_TRY(cudaMemcpy(b4.data(), s->bvh4, sizeof(float4) * 8 * m, cudaMemcpyDeviceToHost));
        RT_CUDA_TRY(cudaMemcpy(root.data(), s->nodes, sizeof(float4) * 4, cudaMemcpyDeviceToHost));
        std::vector<int2> ch(m);
        {
            struct Item { int64_t P, l, r, g; };
            std::vector<Item> st;
            int g0;
            memcpy(&g0, &root[3].w, 4);
            st.push_back({0, 0, n - 1, g0});
            while (!st.empty()) {
                const Item it = st.back();
                st.pop_back();
                if (it.g < it.l || it.g >= it.r || it.g >= m) {
                    rt_set_error("corrupt BVH: split %lld outside node range [%lld, %lld]", (long long)it.g,
                                 (long long)it.l, (long long)it.r);
                    return RT_ECUDA;
                }
                int2 c;
                if (it.l == it.g) {
                    c.x = ~(int)it.l;
                } else {
                    c.x = (int)it.g;
                    int gl;
                    memcpy(&gl, &b4[8 * it.g + 1].w, 4);
                    st.push_back({it.g, it.l, it.g, gl});
                }
                if (it.g + 1 == it.r) {
                    c.y = ~(int)it.r;
                } else {
                    c.y = (int)(it.g + 1);
                    int gr;
                    memcpy(&gr, &b4[8 * it.g + 5].w, 4);
                    st.push_back({it.g + 1, it.g + 1, it.r, gr});
                }
                ch[it.P] = c;
            }
        }
        if (child) memcpy(child, ch.data(), 8 * m);
        std::vector<int32_t> par(2 * n - 1, -1);
        for (int64_t p = 0; p < m; ++p) {
            const int cl = ch[p].x, cr = ch[p].y;
            par[cl < 0 ? m + ~cl : cl] = (int32_t)p;
            par[cr < 0 ? m + ~cr : cr] = (int32_t)p;
        }
        if (parent) memcpy(parent, par.data(), 4 * (2 * n - 1));
        if (boxes) {
            for (int64_t p = 0; p < m; ++p) {
                float* b = boxes + 12 * p;
                if (p == 0) {
                    const float4* q = root.data();
                    b[0] = q[0].x; b[1] = q[0].z; b[2] = q[2].x; b[3] = q[0].y; b[4] = q[0].w; b[5] = q[2].y;
                    b[6] = q[1].x; b[7] = q[1].z; b[8] = q[2].z; b[9] = q[1].y; b[10] = q[1].w; b[11] = q[2].w;
                    continue;
                }
                const int q = par[p];
                const int side = ch[q].y == (int)p ? 1 : 0;
                const int gq = ch[q].x < 0 ? ~ch[q].x : ch[q].x;       // split of Q = right end of its left child
                const float4* h = &b4[8 * (int64_t)gq + 4 * side];
                b[0] = h[0].x; b[1] = h[0].y; b[2] = h[0].z; b[3] = h[1].x; b[4] = h[1].y; b[5] = h[1].z;
                b[6] = h[2].x; b[7] = h[2].y; b[8] = h[2].z; b[9] = h[3].x; b[10] = h[3].y; b[11] = h[3].z;
            }
        }
        if (heights) {
            // subtree heights in reverse breadth-first order (children before parents)
            std::vector<int64_t> bfs;
            bfs.reserve(m);
            bfs.push_back(0);
            for (size_t k = 0; k < bfs.size(); ++k) {
                const int2 c2 = ch[bfs[k]];
                if (c2.x >= 0) bfs.push_back(c2.x);
                if (c2.y >= 0) bfs.push_back(c2.y);
            }
            std::vector<int32_t> hh(m, 0);
            for (size_t k = bfs.size(); k-- > 0;) {
                const int64_t p = bfs[k];
                const int2 c2 = ch[p];
                const int a = c2.x >= 0 ? hh[c2.x] : 0, bb = c2.y >= 0 ? hh[c2.y] : 0;
                hh[p] = 1 + (a > bb ? a : bb);
            }
            memcpy(heights, hh.data(), 4 * m);
        }
    }
    if (cbounds || inv_ext) {
        float cb[9];
        RT_CUDA_TRY(cudaMemcpy(cb, s->cbounds, sizeof cb, cudaMemcpyDeviceToHost));
        if (cbounds) memcpy(cbounds, cb, 6 * sizeof(float));
        if (inv_ext) memcpy(inv_ext, cb + 6, 3 * sizeof(float));
    }
    // the unsorted keys are overwritten by the sort's ping-pong; recompute them on request
    if (morton) {
        rt_set_error("unsorted Morton keys are not retained after the sort");
        return RT_EINVAL;
    }
    return RT_OK;
}

int rt_trace_closest(rt_ctx* c, rt_scene* s, int64_t n, const float* rays, float* hits, uint32_t ray_mask,
                     uint32_t* stats, int32_t flags) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "ctx/scene is NULL");
    RT_CHECK_ARG(n >= 0 && (n == 0 || (rays && hits)), "bad ray/hit buffers");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    RT_CUDA_TRY(cudaSetDevice(c->device));
    return rt_trace_impl(c, s, n, rays, reinterpret_cast<float4*>(hits), ray_mask, stats, flags & RT_TRACE_NO_CUSTOM);
}

// accel.py:1128-1156 with the reference's host dtypes through the chunked
// three-stream pipeline of hostio.cuh: H2D(f64) -> pack -> trace -> expand -> D2H(f64)
int rt_closest_hit_host(rt_ctx* c, rt_scene* s, int64_t n, const double* o, const double* d, const double* tmin,
                        const double* tmax, double tmin_s, double tmax_s, uint32_t ray_mask, double* t,
                        int64_t* inst, int64_t* prim, double* u, double* v, double* nrm, int64_t* stats,
                        int32_t flags) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "ctx/scene is NULL");
    RT_CHECK_ARG(n >= 0, "negative ray count");
    RT_CHECK_ARG(n == 0 || (o && d && t && inst && prim && u && v && nrm), "NULL ray or output buffer");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    if (n == 0) return RT_OK;
    RT_CUDA_TRY(cudaSetDevice(c->device));
    const HostIo in{o, d, tmin, tmax, tmin_s, tmax_s};
    // hits: (t, id, u, v) 16 B + stats 8 B; out: t, inst, prim, u, v (8 B each), normal 24 B, stats 16 B
    auto kernels = [&](const IoSlot& S, int64_t m) -> int {
        float4* hits = (float4*)S.hits;
        uint32_t* st = stats ? (uint32_t*)((char*)S.hits + 16 * m) : nullptr;
        int rc = rt_trace_impl(c, s, m, S.rays, hits, ray_mask, st, flags & RT_TRACE_NO_CUSTOM);
        if (rc) return rc;
        char* O = (char*)S.out;
        return rt_expand_hits_f64(c, s, m, hits, (double*)O, (int64_t*)(O + 8 * m), (int64_t*)(O + 16 * m),
                                  (double*)(O + 24 * m), (double*)(O + 32 * m), (double*)(O + 40 * m), S.rays, st,
                                  (int64_t*)(O + 64 * m), S.o, S.d, tmin ? S.tmin : nullptr,
                                  tmax ? S.tmax : nullptr, tmin_s, tmax_s);
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
    int rc = rt_io_run(c, n, in, 24, 80, kernels, download);
    if (rc) return rc;
    return rt_check_device_error(c);
}

int rt_trace_any(rt_ctx* c, rt_scene* s, int64_t n, const float* rays, uint8_t* hit, uint32_t ray_mask,
                 int32_t flags) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "ctx/scene is NULL");
    RT_CHECK_ARG(n >= 0 && (n == 0 || (rays && hit)), "bad ray/hit buffers");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    RT_CUDA_TRY(cudaSetDevice(c->device));
    return rt_trace_any_impl(c, s, n, rays, hit, ray_mask, flags & RT_TRACE_NO_CUSTOM);
}

// accel.py:1159-1174 any_hit_batch with host float64 rays -> host bool (uint8), same pipeline
int rt_any_hit_host(rt_ctx* c, rt_scene* s, int64_t n, const double* o, const double* d, const double* tmin,
                    const double* tmax, double tmin_s, double tmax_s, uint32_t ray_mask, uint8_t* out,
                    int32_t flags) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "ctx/scene is NULL");
    RT_CHECK_ARG(n >= 0, "negative ray count");
    RT_CHECK_ARG(n == 0 || (o && d && out), "NULL ray or output buffer");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    if (n == 0) return RT_OK;
    RT_CUDA_TRY(cudaSetDevice(c->device));
    const HostIo in{o, d, tmin, tmax, tmin_s, tmax_s};
    auto kernels = [&](const IoSlot& S, int64_t m) -> int {
        return rt_trace_any_impl(c, s, m, S.rays, (uint8_t*)S.out, ray_mask, flags & RT_TRACE_NO_CUSTOM);
    };
    auto download = [&](const IoSlot& S, int64_t b, int64_t m, cudaStream_t so) -> int {
        RT_CUDA_TRY(cudaMemcpyAsync(out + b, S.out, m, cudaMemcpyDeviceToHost, so));
        return RT_OK;
    };
    int rc = rt_io_run(c, n, in, 0, 1, kernels, download);
    if (rc) return rc;
    return rt_check_device_error(c);
}

// world-space emissive triangles for next-event estimation (scene.py:58-76 light rows):
// rows of 16 floats = v0 (3), v1 (3), v2 (3), unit normal (3), emission (3), area
int rt_scene_set_lights(rt_ctx* c, rt_scene* s, int32_t n_lights, const float* rows) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && n_lights >= 0 && (n_lights == 0 || rows), "bad light table");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_free(s->lights, s->stream);
    s->lights = nullptr;
    s->n_lights = n_lights;
    if (n_lights == 0) return RT_OK;
    std::vector<float4> L(5 * (size_t)n_lights);
    for (int k = 0; k < n_lights; ++k) {
        const float* r = rows + 16 * k;
        L[5 * k + 0] = make_float4(r[0], r[1], r[2], r[15]);
        L[5 * k + 1] = make_float4(r[3], r[4], r[5], 0.f);
        L[5 * k + 2] = make_float4(r[6], r[7], r[8], 0.f);
        L[5 * k + 3] = make_float4(r[9], r[10], r[11], 0.f);
        L[5 * k + 4] = make_float4(r[12], r[13], r[14], 0.f);
    }
    RT_CUDA_TRY(rt_alloc((void**)&s->lights, sizeof(float4) * L.size(), s->stream));
    RT_CUDA_TRY(cudaMemcpy(s->lights, L.data(), sizeof(float4) * L.size(), cudaMemcpyHostToDevice));
    return RT_OK;
}

int rt_scene_set_spheres(rt_ctx* c, rt_scene* s, int32_t n_spheres, const double* rows) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && n_spheres >= 0 && (n_spheres == 0 || rows), "bad sphere table");
    RT_CHECK_ARG(n_spheres <= s->n, "more spheres than primitives");
    for (int k = 0; k < n_spheres; ++k)
        RT_CHECK_ARG(rows[16 * k + 15] > 0.0, "sphere radius must be > 0");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_free(s->spheres, s->stream);
    s->spheres = nullptr;
    s->n_spheres = n_spheres;
    if (n_spheres == 0) return RT_OK;
    RT_CUDA_TRY(rt_alloc((void**)&s->spheres, sizeof(double) * 16 * (size_t)n_spheres, s->stream));
    RT_CUDA_TRY(cudaMemcpy(s->spheres, rows, sizeof(double) * 16 * (size_t)n_spheres, cudaMemcpyHostToDevice));
    return RT_OK;
}

static int render_args(rt_ctx* c, rt_scene* s, const rt_render_params* p) {
    RT_CHECK_ARG(p->width >= 1 && p->height >= 1 && p->s1 > p->s0 && p->s0 >= 0,
                 "width, height, and spp must all be >= 1");
    RT_CHECK_ARG(p->integrator == RT_INTEG_EYE || p->integrator == RT_INTEG_AO || p->integrator == RT_INTEG_PT ||
                     p->integrator == RT_INTEG_PTNEE,
                 "integrator must be eye, ao, pt or pt-nee");
    RT_CHECK_ARG(p->kernel == RT_KERNEL_MEGA || p->integrator == RT_INTEG_EYE || p->integrator == RT_INTEG_PT,
                 "ao and pt-nee run in the megakernel (kernel=mega)");
    RT_CHECK_ARG(p->integrator != RT_INTEG_AO || (p->ao_count >= 1 && p->ao_length > 0.0f), "bad ao parameters");
    RT_CHECK_ARG(p->integrator != RT_INTEG_PTNEE || s->n_lights > 0, "pt-nee needs a light table");
    RT_CHECK_ARG(p->max_depth >= 1, "max_depth must be >= 1");
    RT_CHECK_ARG(p->kernel == RT_KERNEL_MEGA || p->kernel == RT_KERNEL_WAVEFRONT, "unknown kernel");
    if (!s->built) { rt_set_error("BVH not built"); return RT_ESTATE; }
    return RT_OK;
}

int rt_render(rt_ctx* c, rt_scene* s, const rt_render_params* p, float* accum, uint64_t* rays_out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && p && accum, "NULL argument");
    int rc = render_args(c, s, p);
    if (rc) return rc;
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rc = rt_render_impl(c, s, p, accum, rays_out);
    if (rc) return rc;
    if (rays_out) return rt_check_device_error(c);
    return RT_OK;
}

int rt_render_host(rt_ctx* c, rt_scene* s, const rt_render_params* p, double* host_out, int32_t n_chunks,
                   uint64_t* rays_out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && p && host_out, "NULL argument");
    RT_CHECK_ARG(n_chunks >= 1, "n_chunks must be >= 1");
    int rc = render_args(c, s, p);
    if (rc) return rc;
    RT_CUDA_TRY(cudaSetDevice(c->device));
    return rt_render_host_impl(c, s, p, host_out, n_chunks, rays_out);
}

int rt_resolve(rt_ctx* c, const float* accum, int64_t npix, int32_t gamma, uint8_t* rgb) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && accum && rgb && npix >= 0, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    int rc = rt_resolve_impl(c, accum, npix, gamma, rgb);
    if (rc) return rc;
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    int e = 0;
    RT_CUDA_TRY(cudaMemcpy(&e, c->d_error, sizeof e, cudaMemcpyDeviceToHost));
    if (e == RT_EINVAL) {
        int z = 0;
        cudaMemcpy(c->d_error, &z, sizeof z, cudaMemcpyHostToDevice);
        rt_set_error("accumulation buffer has pixels with zero samples");
        return RT_EINVAL;
    }
    return rt_check_device_error(c);
}

int rt_raygen(rt_ctx* c, const rt_render_params* p, int32_t sample, float* rays) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && p && rays, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    return rt_raygen_impl(c, p, sample, rays);
}

}  // extern "C"
