// rt_common.cuh -- shared device helpers for librt_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/rt_b200.h"

#define RT_FULL 0xFFFFFFFFu
#define RT_STACK 64                // traversal stack entries (== MAX_STACK_DEPTH, accel.py:44)
#define RT_SENTINEL 0x7FFFFFFF     // bottom-of-stack marker (never a node or leaf id)

// --------------------------------------------------------------------------
// context / scene
// --------------------------------------------------------------------------
struct rt_ctx {
    int device;
    int num_sms;
    cudaStream_t own_stream;
    cudaStream_t stream;
    cudaEvent_t ev0, ev1;
    cudaEvent_t prof[8];           // stage events for rt_bvh_build_profiled
    int profiling;
    // pinned staging + device scratch for rt_closest_hit_host
    void* h_stage;                 // rt_h2d: two pinned 16-MB chunks for pageable sources
    size_t h_stage_bytes;
    cudaEvent_t stage_ev[2];
    void* d_stage;
    size_t d_stage_bytes;
    unsigned int* d_counter;       // persistent-kernel work counters (64 slots)
    int* d_error;                  // device-side error flag
    void* d_probe;                 // tile-probe heavy queue + claims of eye renders (render.cu), grown on demand
    int64_t probe_tiles;
    unsigned probe_epoch;          // claim tag of the last probed render
    const void* lp_scene;          // the last probe-capable eye frame: scene and tile geometry
    int64_t lp_key[4];             // (a replay of its heavy-tile queue needs the same ones)
    void* d_chunk_done;            // per-tile finished sample chunks of chunked PT frames (render.cu)
    int64_t chunk_tiles;
    void* d_rb;                    // rt_render_host: float64 rows + fp32 sums of a frame
    int64_t rb_pix;                // pixels d_rb holds
    void* h_tab;                   // pinned staging of rt_scene_compile's small tables (mesh.cu)
    size_t h_tab_bytes;
    cudaEvent_t tab_ev;            // its last copies (the buffer is rewritten only after them)
    // host-buffer transfer pipeline (hostio.cuh): copy-in / copy-out streams + events
    cudaStream_t io_in, io_out;
    cudaEvent_t io_ev[9];
    void* d_io;
    size_t d_io_bytes;
    // every entry point taking the context holds this lock: the staging slots, work counters
    // and error flag are per context, so calls on one device from several host threads
    // (ctypes releases the GIL) are serialised instead of racing
    std::recursive_mutex* mu;
};

struct rt_scene {
    unsigned* probe_hint;  // device word: the last probed eye frame of this scene stopped probing (render.cu)
    int64_t n;
    int n_mat;
    int device;
    cudaStream_t stream;  // storage is stream-ordered pool memory, freed on this stream
    int mask_uniform;     // every primitive has instance mask `mask_value` (the build skips the gather)
    uint32_t mask_value;
    // inputs (resident)
    float* tris;          // (n, 9) world vertices
    float4* tri_attr;     // (n) normal.xyz, material id bits   (F9 normals)
    int32_t* tri_inst;    // (n)
    int32_t* tri_prim;    // (n)
    uint32_t* tri_mask;   // (n)
    float4* mat_color;    // (n_mat)
    float4* mat_emissive; // (n_mat)
    // LBVH
    int built;
    int bits;
    float4* nodes;        // root record, 4 float4: root child boxes, child ids, tree height, BVH4 root
    float4* tri_sorted;   // (n, 3) leaf-ordered vertices; v0.w = flat id, v1.w = mask
    float4* bvh4;         // (max(n-1,1), 8) 4-wide traversal view (grandchildren of each binary node)
    // build scratch
    void* keys_a; void* keys_b;     // u32 or u64 Morton keys
    uint32_t* vals_a; uint32_t* vals_b;
    int2* child;                    // (n-1) Karras child ids (parents, boxes, heights derived on download)
    unsigned int* flags;            // (n-1) global split slots of the emit climb
    float* cbounds;                 // 6 floats + 3 inv_ext (+pad)
    unsigned int* sort_scratch;     // hist + counters + look-back status
    size_t sort_scratch_words;
    float4* leaf_box;               // global split-slot boxes (4 float4 per split)
    float4* lights;                 // (n_lights, 5): (v0, area), v1, v2, normal, emission
    int n_lights;
    void* emit_items;               // boundary-crossing nodes handed from emit phase A to phase B
    unsigned int* seg_count;        // per emit block: items in its segment
    // custom primitives: the last n_spheres flat primitives are spheres
    double* spheres;                // (n_spheres, 16): inverse 3x4, center, radius
    int n_spheres;
    // as a bottom-level structure of a two-level rt_tlas (tlas.cu)
    double* lnormal64;              // (n, 3) float64 local normals (reference order), triangles
    double* lrows64;                // (n, 9) float64 local vertices (BLAS): the host query's exact refinement
    double* wnormal64;              // (n, 3) float64 world normals (flat scene, nullable): host query output
    double* inst_inv64;             // (instances, 12) float64 inverses of a flat scene (nullable): with
                                    // lrows64 = the local vertices per flat id, the query refines in local space
    int custom;                     // 1: prims are AABBs of custom primitives (geom_type, data_offset)
    int geom_type;
    int64_t data_offset;
};

// --------------------------------------------------------------------------
// error plumbing
// --------------------------------------------------------------------------
void rt_set_error(const char* fmt, ...);
#define RT_CUDA_TRY(expr)                                                        \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) {                                                  \
            rt_set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),  \
                         __FILE__, __LINE__);                                     \
            return RT_ECUDA;                                                      \
        }                                                                         \
    } while (0)

#define RT_CTX_LOCK(ctx)                                                   \
    if (!(ctx)) {                                                          \
        rt_set_error("ctx is NULL");                                       \
        return RT_EINVAL;                                                  \
    }                                                                      \
    std::lock_guard<std::recursive_mutex> _rt_ctx_guard(*(ctx)->mu)

#define RT_CHECK_ARG(cond, msg)              \
    do {                                     \
        if (!(cond)) {                       \
            rt_set_error("%s", msg);         \
            return RT_EINVAL;                \
        }                                    \
    } while (0)

// Scene / mesh storage comes from the device's stream-ordered memory pool (its release
// threshold is raised at context creation, so freed blocks stay cached and compiling a
// scene again costs no cudaMalloc / cudaFree).  rt_alloc synchronises the stream once the
// allocation is enqueued, so the block is usable from any stream afterwards.
inline cudaError_t rt_alloc(void** p, size_t bytes, cudaStream_t st, bool sync = true) {
    cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, st);
    if (e == cudaSuccess && sync) e = cudaStreamSynchronize(st);
    return e;
}
inline void rt_free(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

// host -> device copy on the context stream; large pageable sources are staged through
// pinned chunks by several host threads (capi.cu)
int rt_h2d(rt_ctx* c, void* dst, const void* src, size_t bytes);

// reads and clears the device error flag (synchronises the context stream)
int rt_check_device_error(rt_ctx* ctx);
// scene storage for n primitives (contents unset) / material table upload
extern "C" int rt_scene_alloc(rt_ctx* c, int64_t n, int32_t n_mat, rt_scene** out);
extern "C" int rt_scene_alloc_ex(rt_ctx* c, int64_t n, int32_t n_mat, rt_scene** out, int sync);
extern "C" int rt_scene_set_materials(rt_ctx* c, rt_scene* s, const float* mat_color, const float* mat_emissive);

// --------------------------------------------------------------------------
// exact fp32 helpers (parity-critical paths use explicit selects, no FMNMX
// NaN/zero-sign ambiguity, no FMA contraction)
// --------------------------------------------------------------------------
__device__ __forceinline__ float sel_min(float a, float b) { return b < a ? b : a; }
__device__ __forceinline__ float sel_max(float a, float b) { return b > a ? b : a; }

// orderable uint encoding of fp32 for atomicMin/atomicMax
__device__ __forceinline__ unsigned int f2ord(float f) {
    unsigned int u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned int u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// --------------------------------------------------------------------------
// PCG32 + splitmix64 streams (sampling.py:38-79), bit-exact
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t rt_mix64(uint64_t z) {
    z = z + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t rt_pcg_next(uint64_t& state, uint64_t inc) {
    uint64_t old = state;
    state = old * 6364136223846793005ull + inc;
    uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return __funnelshift_r(xs, xs, rot);   // rotate right
}
// the per-pixel part of the stream hash, mix(mix(seed) ^ pix): computed once per pixel by
// callers that draw several samples of it
__device__ __forceinline__ uint64_t rt_stream_pixel(uint64_t seed, uint64_t pix) {
    return rt_mix64(rt_mix64(seed) ^ pix);
}
__device__ __forceinline__ void rt_stream_from_pixel(uint64_t hp, uint64_t s, uint64_t& state, uint64_t& inc) {
    uint64_t h = rt_mix64(hp ^ s);
    inc = (rt_mix64(h ^ 0xDA3E39CB94B95BDBull) << 1) | 1ull;
    state = 0;
    rt_pcg_next(state, inc);
    state += h;
    rt_pcg_next(state, inc);
}
__device__ __forceinline__ void rt_stream_for(uint64_t seed, uint64_t pix, uint64_t s, uint64_t& state,
                                              uint64_t& inc) {
    uint64_t h = rt_mix64(rt_mix64(rt_mix64(seed) ^ pix) ^ s);
    inc = (rt_mix64(h ^ 0xDA3E39CB94B95BDBull) << 1) | 1ull;
    state = 0;
    rt_pcg_next(state, inc);
    state += h;
    rt_pcg_next(state, inc);
}
// u32 * 2^-32 in [0, 1): round toward zero so 2^32-1 never rounds up to 1.0f
__device__ __forceinline__ float rt_uniform(uint64_t& state, uint64_t inc) {
    return __uint2float_rz(rt_pcg_next(state, inc)) * 0x1p-32f;
}

// --------------------------------------------------------------------------
// ray / hit records
// --------------------------------------------------------------------------
struct TraceRay {
    float ox, oy, oz, tmin, dx, dy, dz, tmax;
};

__device__ __forceinline__ TraceRay load_ray(const float* rays, int64_t i) {
    const float4* r = reinterpret_cast<const float4*>(rays) + 2 * i;
    float4 a = __ldg(r), b = __ldg(r + 1);
    TraceRay R;
    R.ox = a.x; R.oy = a.y; R.oz = a.z; R.tmin = a.w;
    R.dx = b.x; R.dy = b.y; R.dz = b.z; R.tmax = b.w;
    return R;
}

// camera.py:81-97 in fp32.  cam = origin, right, up, forward, distortion
__device__ __forceinline__ bool rt_primary_dir(const float* cam, float u, float v, float& dx, float& dy,
                                               float& dz) {
    float su = 2.0f * u - 1.0f, sv = 1.0f - 2.0f * v;
    float px = cam[3] * su + cam[6] * sv;
    float py = cam[4] * su + cam[7] * sv;
    float pz = cam[5] * su + cam[8] * sv;
    float c = cam[12] * (px * px + py * py + pz * pz);
    float denom = 1.0f + c;
    if (denom <= 0.0f) { dx = dy = dz = 0.0f; return false; }
    dx = cam[9] + px / denom;
    dy = cam[10] + py / denom;
    dz = cam[11] + pz / denom;
    float inv = 1.0f / sqrtf(dx * dx + dy * dy + dz * dz);
    dx *= inv; dy *= inv; dz *= inv;
    return true;
}

#define RT_PROF(ctx, k) do { if ((ctx)->profiling) cudaEventRecord((ctx)->prof[k], (ctx)->stream); } while (0)

// host-side launch helpers (defined in capi.cu / lbvh.cu / trace.cu / render.cu)
int rt_lbvh_build_impl(rt_ctx* ctx, rt_scene* s, int bits);
// custom_mode: 0 = spheres intersected, 1 = reaching one is RT_EUNSUPPORTED (no intersector registered)
int rt_trace_impl(rt_ctx* ctx, rt_scene* s, int64_t n, const float* rays, float4* hits, uint32_t mask,
                  uint32_t* stats, int custom_mode);
int rt_trace_any_impl(rt_ctx* ctx, rt_scene* s, int64_t n, const float* rays, uint8_t* out, uint32_t mask,
                      int custom_mode);
int rt_expand_hits_f64(rt_ctx* ctx, rt_scene* s, int64_t n, const float4* hits, double* t, int64_t* inst,
                       int64_t* prim, double* u, double* v, double* nrm, const float* rays, const uint32_t* st32,
                       int64_t* st64, const double* o64 = nullptr, const double* d64 = nullptr,
                       const double* tmin64 = nullptr, const double* tmax64 = nullptr, double tmin_s = 0.0,
                       double tmax_s = 0.0);
int rt_pack_rays_f64(rt_ctx* ctx, int64_t n, const double* o, const double* d, const double* tmin,
                     const double* tmax, float* rays);
int rt_render_impl(rt_ctx* ctx, rt_scene* s, const rt_render_params* p, float* accum, uint64_t* rays_out,
                   double* out64 = nullptr);
int rt_render_host_impl(rt_ctx* ctx, rt_scene* s, const rt_render_params* p, double* host_out, int n_chunks,
                        uint64_t* rays_out);
int rt_io_streams(rt_ctx* c);
int rt_raygen_impl(rt_ctx* ctx, const rt_render_params* p, int sample, float* rays);
int rt_resolve_impl(rt_ctx* ctx, const float* accum, int64_t npix, int gamma, uint8_t* rgb);
