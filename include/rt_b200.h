/*
 * rt_b200.h -- C ABI of the B200-native ray-tracing hot path (librt_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as void*).  Every entry point returns 0 on success or a
 * negative RT_E* code; rt_last_error() holds a thread-local message.
 *
 * The reference (pkg/src/pathtrace) is a Python/numba library with no FFI;
 * each entry point below replaces the reference function named beside it and
 * is bound from Python through ctypes (paper_2603_00292_b200/_native.py; the
 * binding a reference maintainer would add is shown in INTEGRATION.md).
 */
#ifndef RT_B200_H
#define RT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RT_OK 0
#define RT_EINVAL (-1)        /* bad argument                 -> ValueError   */
#define RT_ECUDA (-2)         /* CUDA runtime failure         -> RuntimeError */
#define RT_EUNSUPPORTED (-3)  /* a ray reached a custom primitive with no intersector -> RegistryError */
#define RT_EDEPTH (-4)        /* BVH deeper than the traversal stack -> BuildError (accel.py:148-149) */
#define RT_ENOMEM (-5)        /* device allocation failed     -> MemoryError  */
#define RT_ESTATE (-6)        /* e.g. trace before build      -> RuntimeError */
#define RT_ENCCL (-7)         /* NCCL failure (rt_multi_render) -> RuntimeError */
#define RT_EBUILD (-8)        /* invalid geometry (Blas.from_mesh checks, accel.py:223-236) -> BuildError */

#define RT_INTEG_EYE 0        /* integrators.py:129-141 _sample_eye   */
#define RT_INTEG_AO 1         /* integrators.py:144-179 _sample_ao    (megakernel) */
#define RT_INTEG_PT 2         /* integrators.py:182-235 _sample_pt    */
#define RT_INTEG_PTNEE 3      /* integrators.py:238-331 _sample_ptnee (megakernel) */

/* trace flags (rt_trace_closest / rt_trace_any / rt_closest_hit_host / rt_any_hit_host) */
#define RT_TRACE_NO_CUSTOM 1  /* no intersector registered for the scene's custom primitives
                                 (registry=None, accel.py:1002-1008): a ray that reaches one
                                 fails with RT_EUNSUPPORTED -> RegistryError (accel.py:800-803) */

#define RT_KERNEL_MEGA 0      /* one persistent kernel per frame (K7)      */
#define RT_KERNEL_WAVEFRONT 1 /* raygen / extend / shade / accumulate (K8) */

typedef struct rt_ctx rt_ctx;
typedef struct rt_scene rt_scene;
typedef struct rt_tlas rt_tlas;
typedef struct rt_mesh rt_mesh;

/* Frame parameters: render_frame(scene, width, height, spp, integrator, seed,
 * workers, cfg, jitter) -- integrators.py:426-473.  Samples [s0, s1) are
 * rendered with the GLOBAL sample index in the per-(seed, pixel, sample)
 * stream hash (sampling.py:67-73), so a sample split across GPUs reproduces
 * the single-GPU random numbers exactly.  Pixels [pix_lo, pix_hi) restrict the
 * frame to a row-major pixel range (tile split); 0/0 means the whole frame. */
typedef struct {
    int32_t width, height;
    int32_t s0, s1;
    uint64_t seed;
    int32_t jitter;
    int32_t integrator;       /* RT_INTEG_EYE | RT_INTEG_PT */
    int32_t max_depth;        /* IntegratorConfig.max_depth (integrators.py:56-74) */
    int32_t kernel;           /* RT_KERNEL_MEGA | RT_KERNEL_WAVEFRONT */
    float cam[13];            /* origin, right, up, forward, distortion (integrators.py:397-402) */
    float sky[3];
    float background[3];
    float normal_offset;      /* 1e-4 * scene diagonal (integrators.py:405-413) */
    int64_t pix_lo, pix_hi;
    /* tile split across GPUs: with a whole-frame pixel range the frame is cut
     * into rows of 8x4-pixel tiles; only tile rows r with r % band_stride ==
     * band_offset are rendered (interleaved bands balance the load).  1/0 = all. */
    int32_t band_stride, band_offset;
    int32_t ao_count;         /* IntegratorConfig.ao_ray_count */
    float ao_length;          /* IntegratorConfig.ao_max_length */
} rt_render_params;

/* ---- context --------------------------------------------------------- */
int rt_ctx_create(int device, rt_ctx** out);
void rt_ctx_destroy(rt_ctx* ctx);
/* all work of the context is issued on this cudaStream_t (used verbatim; NULL =
 * the legacy default stream); a new context uses its own non-blocking stream */
int rt_ctx_set_stream(rt_ctx* ctx, void* cuda_stream);
int rt_ctx_sync(rt_ctx* ctx);
/* the context's 64 device work counters after the last launch (diagnostics: [0] work units
 * taken by the persistent kernels, [32..33] closest-hit queries of the last render (u64)) */
int rt_ctx_counters(rt_ctx* ctx, uint32_t* out64);
/* tile-probe scheduling of megakernel eye renders (process-wide; render.cu): before
 * rendering, one ray per 8x4 tile walks under a budget of walk steps and tiles that run out
 * are rendered first.  0 disables it (row-major tiles); the default is 24 or the
 * RT_PROBE_BUDGET environment variable.  The frame is identical either way: only the order
 * in which tiles are rendered changes. */
int rt_set_probe_budget(int32_t budget, int32_t* previous);
/* the last probed eye render of the context: out4 = {tiles probed (batch-rounded), heavy
 * tiles queued, queue pops, 1 + first tile past the probe when probing stopped early (0:
 * it did not)} */
int rt_probe_stats(rt_ctx* ctx, uint32_t* out4);
int rt_device_count(int* n);
const char* rt_last_error(void);
const char* rt_version(void);

/* ---- scene (replaces compile_scene's geometry side, scene.py:79-141; the
 *      instances are flattened to world-space triangles on the host) ------ */
/* tris: (n, 9) fp32 world vertices, host.  normals: (n, 3) fp32 world normal per
 * triangle computed reference-style (local cross, inverse-transpose, accel.py:843-847).
 * tri_inst / tri_prim: (n,) owning instance and primitive index; tri_mask: (n,) the
 * instance visibility mask; tri_material: (n,) material row.  mat_color /
 * mat_emissive: (n_mat, 3).  Triangle ids must be ordered by (inst, prim) so the
 * reference tie rule (accel.py:629, 815-817) becomes "lowest flat id". */
int rt_scene_create(rt_ctx* ctx, int64_t n, const float* tris, const float* normals,
                    const int32_t* tri_inst, const int32_t* tri_prim, const uint32_t* tri_mask,
                    const int32_t* tri_material, const float* mat_color, const float* mat_emissive,
                    int32_t n_mat, rt_scene** out);
void rt_scene_destroy(rt_scene* scene);
/* custom primitives (compile_scene's sphere instances, scene.py:101-112): the LAST
 * n_spheres primitives of the scene are spheres, each its own instance.  Their rows
 * in rt_scene_create's `tris` hold the instance's world AABB as (lo, hi, lo) so the
 * LBVH bounds them like triangles; `rows` holds 16 doubles per sphere: the instance
 * inverse 3x4 (row-major, accel.py:311-336), the local center xyz and the radius.
 * Hits on them are computed in float64 (geometry.py:334-363) with u = v = 0. */
int rt_scene_set_spheres(rt_ctx* ctx, rt_scene* scene, int32_t n_spheres, const double* rows);
/* new vertex positions for the same triangles (Blas.refit(vertices), accel.py:263-283);
 * host (n, 9) fp32, copied on the context stream; the BVH must be rebuilt */
int rt_scene_set_vertices(rt_ctx* ctx, rt_scene* scene, const float* tris);

/* Device-side refit from the reference's own input (Blas.refit(vertices), accel.py:263-283):
 * an indexed mesh whose faces stay resident on the device, instanced into the flat scene
 * at n_inst triangle offsets.  xform: n_inst rows of 21 doubles = the instance 3x4 matrix
 * (row-major, accel.py:311-336) then the 3x3 block of its inverse (row-major).
 * rt_scene_refit_mesh uploads the vertices (nv, 3) (the count fixed at create) as float64,
 * or as fp32 when vertices_f32 != 0 (widened exactly on the device), then one kernel writes
 * every instance's world triangles (fp32) and world normals exactly as compile_scene does
 * on the host (float64, reference operation order, no FMA; normals per accel.py:843-847
 * from the local geometry.py:229-237 normal).  The BVH must be rebuilt. */
#define RT_MESH_LOCAL 1   /* a BLAS (two-level Blas.refit): one placement at offset 0, rows = the local
                             vertices, float64 local normals into rt_scene_set_local_normals' array */
int rt_mesh_create(rt_ctx* ctx, int64_t n_vertices, int64_t n_faces, const int32_t* faces, int32_t n_inst,
                   const double* xform, const int64_t* tri_offset, int32_t flags, rt_mesh** out);
int rt_scene_refit_mesh(rt_ctx* ctx, rt_scene* scene, rt_mesh* mesh, int64_t n_vertices, const void* vertices,
                        int32_t vertices_f32);
void rt_mesh_destroy(rt_mesh* mesh);
/* ---- compile_scene on the device (scene.py:79-141) ----------------------
 * rt_mesh_upload: one mesh as the reference holds it -- vertices (nv, 3) float64 and faces
 * (nf, 3) int64, host -- goes up once and is validated on the device exactly like
 * Blas.from_mesh (accel.py:223-236): zero faces -> "cannot build over zero primitives",
 * an index outside [0, nv) -> "face index out of range", else the first triangle with a
 * non-finite coordinate -> "non-finite bounds for primitive k" (all RT_EBUILD).  bounds6
 * receives the float64 root box (lo xyz, hi xyz: the union of the triangle boxes, i.e. the
 * reference Blas's root node bounds).  The mesh stays resident (faces as int32) for
 * rt_scene_compile and later rt_scene_refit_mesh calls. */
int rt_mesh_upload(rt_ctx* ctx, int64_t n_vertices, const double* vertices, int64_t n_faces, const int64_t* faces,
                   double* bounds6, rt_mesh** out);
/* rt_mesh_upload in two halves: _async enqueues the copies and the validation on the
 * context stream and returns the mesh (argument errors and zero faces are reported here);
 * the host arrays must stay valid until _finish, which reads the verdict back (the same
 * RT_EBUILD errors; the caller then destroys the mesh) and fills bounds6.  rt_scene_compile
 * (and rt_bvh_build after it) may be called between the two: their kernels run behind the
 * validation on the stream and the compile writes nothing for a mesh that fails it; the scene is usable only after every one of its
 * meshes finished successfully (a mesh whose _finish failed is refused, RT_ESTATE): that
 * _finish also synchronises the stream the scene was allocated on. */
int rt_mesh_upload_async(rt_ctx* ctx, int64_t n_vertices, const double* vertices, int64_t n_faces,
                         const int64_t* faces, rt_mesh** out);
int rt_mesh_upload_finish(rt_ctx* ctx, rt_mesh* mesh, double* bounds6);
int rt_mesh_info(rt_mesh* mesh, int64_t* n_vertices, int64_t* n_faces, double* bounds6);
/* one instance of compile_scene (Instance(blas_of_mesh[decl.mesh], decl.frame, decl.mask),
 * scene.py:91-97): matrix = frame_to_matrix(frame), inverse = invert_affine(matrix), both 3x4
 * row-major float64 (accel.py:311-336) */
typedef struct {
    int32_t mesh;             /* index into the meshes array */
    int32_t material;         /* material row */
    uint32_t mask;            /* instance visibility mask */
    int32_t reserved;
    double matrix[12];
    double inverse[12];
} rt_instance_src;
/* one custom primitive (a sphere instance, scene.py:101-112): its instance world AABB rounded
 * outward to fp32 as (lo, hi, lo); row = instance inverse 3x4, local center xyz, radius */
typedef struct {
    float box[9];
    int32_t material;
    uint32_t mask;
    double row[16];
} rt_custom_src;
/* The flat scene of all instances in instance order (flat id = (instance, prim) order, so the
 * reference tie rule is "lowest flat id"), written on the device by one kernel per mesh:
 * world fp32 rows (m . v in float64, reference operation order), float64 world normals
 * (geometry.py:229-237 local normal, accel.py:843-847 inverse-transpose), the float64 local
 * rows + instance inverses of the host query's refinement, ids, masks, materials; custom
 * primitives appended.  Every mesh referenced keeps its placements for rt_scene_refit_mesh.
 * The BVH is not built (rt_bvh_build). */
int rt_scene_compile(rt_ctx* ctx, int32_t n_meshes, rt_mesh* const* meshes, int32_t n_inst,
                     const rt_instance_src* instances, int32_t n_custom, const rt_custom_src* custom,
                     const float* mat_color, const float* mat_emissive, int32_t n_mat, rt_scene** out);
/* the scene's per-primitive ids, device -> host (any pointer may be NULL; synchronises) */
int rt_scene_get_ids(rt_ctx* ctx, rt_scene* scene, int32_t* tri_inst, int32_t* tri_prim, uint32_t* tri_mask,
                     int32_t* tri_material);
/* a render replica of a built scene on dst's device (multi-GPU render_frame): geometry,
 * shading tables and the built LBVH copied device to device (no host-query extras) */
int rt_scene_clone(rt_ctx* src, rt_scene* scene, rt_ctx* dst, rt_scene** out);
/* the scene's geometry, device -> host (parity checks; any pointer may be NULL): (n, 9) fp32
 * rows, (n, 3) fp32 shading normals, (n, 3) float64 world normals, (n, 9) float64 local rows */
int rt_scene_get_geometry(rt_ctx* ctx, rt_scene* scene, float* tris9, float* normals3, double* normals64,
                          double* local_rows9);
/* world normals of the scene's triangles recomputed on the device from its current (world)
 * vertices, float64 in the reference order with an identity frame (after
 * rt_scene_set_vertices, whose rows are world triangles) */
int rt_scene_update_normals(rt_ctx* ctx, rt_scene* scene);
/* float64 world normals of a flat scene, (n, 3) (optional): the host query returns them
 * as they are (compile_scene's reference-style float64 normals) instead of the fp32 copy
 * used for shading; device refits keep them current */
int rt_scene_set_normals64(rt_ctx* ctx, rt_scene* scene, const double* normals);
/* a flat scene's instance inverses (n_inst, 12: 3x4 row-major) and the float64 LOCAL vertices
 * of every flat primitive (n, 9) (optional): the host query then recomputes each hit's
 * (t, u, v) along the reference's own path (local ray, _tri_hit on local vertices).
 * rt_scene_update_normals (new world rows) drops them; Scene.refit_mesh keeps them current. */
int rt_scene_set_local_frames(rt_ctx* ctx, rt_scene* scene, int32_t n_inst, const double* inv12, const double* rows);
/* the scene's current (n, 9) fp32 triangle rows, device -> host (synchronises) */
int rt_scene_get_vertices(rt_ctx* ctx, rt_scene* scene, float* tris);

/* ---- LBVH build (replaces _build_bvh, accel.py:68-187; K1-K5) ---------- */
/* morton_bits: 30 or 63.  build_ms (nullable): device time of the build
 * (CUDA events on the context stream; synchronises). */
int rt_bvh_build(rt_ctx* ctx, rt_scene* scene, int morton_bits, float* build_ms);
/* same build with CUDA events between stages: stage_ms[6] = bounds, morton,
 * histogram, radix passes, split-slot init, fused karras+refit+leaf gather (device ms) */
int rt_bvh_build_profiled(rt_ctx* ctx, rt_scene* scene, int morton_bits, float* stage_ms);
/* root box (6), tree height (stack bound) and node count */
int rt_bvh_info(rt_ctx* ctx, rt_scene* scene, float* root6, int32_t* height, int64_t* n_internal);
/* parity download; every pointer nullable.  sorted_keys (n) u64, order (n) u32,
 * child (n-1, 2) i32 (>=0 internal, <0 = ~leaf), parent (2n-1) i32,
 * boxes (n-1, 12) f32 [lo_L hi_L lo_R hi_R], heights (n-1) i32,
 * centroid_bounds (6) f32, inv_ext (3) f32, morton (n) u64 unsorted keys */
int rt_bvh_download(rt_ctx* ctx, rt_scene* scene, uint64_t* sorted_keys, uint32_t* order,
                    int32_t* child, int32_t* parent, float* boxes, int32_t* heights,
                    float* centroid_bounds, float* inv_ext, uint64_t* morton);

/* ---- closest hit (replaces _closest_batch / closest_hit_batch, accel.py:950-976, 1128-1156; K6) */
/* Device buffers.  rays: (n, 8) f32 [ox oy oz tmin dx dy dz tmax];
 * hits: (n, 4) [t (f32), flat id (i32, -1 miss), u, v]; stats (nullable): (n, 2)
 * u32 [triangle tests, node visits]. */
int rt_trace_closest(rt_ctx* ctx, rt_scene* scene, int64_t n, const float* rays, float* hits,
                     uint32_t ray_mask, uint32_t* stats, int32_t flags);
/* Host buffers with the reference's dtypes (float64 / int64), in chunks through a
 * three-stream pipeline (H2D of chunk k+1 || kernels of chunk k || D2H of chunk k-1;
 * full-rate DMA when the host buffers are pinned).  t_min / t_max: per-ray arrays, or
 * NULL to broadcast the scalars t_min_s / t_max_s (the reference's defaults 0, 1e30).
 * Misses: t = -1, inst = prim = -1 (accel.py:964, 1144).  stats nullable (n, 2) int64. */
int rt_closest_hit_host(rt_ctx* ctx, rt_scene* scene, int64_t n, const double* origins,
                        const double* dirs, const double* t_min, const double* t_max, double t_min_s,
                        double t_max_s, uint32_t ray_mask, double* t, int64_t* inst, int64_t* prim,
                        double* u, double* v, double* normal, int64_t* stats, int32_t flags);

/* ---- any hit (replaces _any_batch / any_hit_batch, accel.py:979-992, 1159-1174) */
/* device rays (n, 8) -> hit (n) uint8 (1 = some accepted intersection in [tmin, tmax]) */
int rt_trace_any(rt_ctx* ctx, rt_scene* scene, int64_t n, const float* rays, uint8_t* hit,
                 uint32_t ray_mask, int32_t flags);
/* host float64 rays -> host uint8 (numpy bool); same pipeline and t-range convention */
int rt_any_hit_host(rt_ctx* ctx, rt_scene* scene, int64_t n, const double* origins, const double* dirs,
                    const double* t_min, const double* t_max, double t_min_s, double t_max_s,
                    uint32_t ray_mask, uint8_t* hit, int32_t flags);
/* emissive triangles for pt-nee (scene.py:58-76): rows of 16 floats =
 * v0, v1, v2, unit normal, emission (3 each), area */
int rt_scene_set_lights(rt_ctx* ctx, rt_scene* scene, int32_t n_lights, const float* rows);

/* ---- render (replaces render_frame / _render_chunk, integrators.py:334-473; K7/K8) */
/* accum: device (H*W, 4) f32 running (r, g, b, n) sums, row 0 on top, added to in
 * place (sample order per pixel).  rays_out (nullable): closest-hit queries issued. */
int rt_render(rt_ctx* ctx, rt_scene* scene, const rt_render_params* p, float* accum,
              uint64_t* rays_out);
/* render_frame in one call (integrators.py:426-473): the frame rendered from zero sums and
 * delivered, synchronously, into host_out = a HOST (H*W, 4) float64 AccumBuffer array
 * (pinned memory for an overlapped copy); pixels outside p's pixel range / band set are 0.
 * The values are the exact float64 widening of the fp32 sums rt_render accumulates.  Eye
 * frames in the megakernel write their float64 rows directly; a whole eye frame with
 * n_chunks > 1 (<= 8, and rays_out NULL) renders in n_chunks row chunks, each copied out
 * while the next renders.  rays_out (nullable): closest-hit queries of the frame. */
int rt_render_host(rt_ctx* ctx, rt_scene* scene, const rt_render_params* p, double* host_out,
                   int32_t n_chunks, uint64_t* rays_out);
/* device resolve (scene_io.py:349-355): accum (npix, 4) f32 running sums -> rgb (npix, 3)
 * uint8, mean clamped to [0, 1], ^(1/2.2) when gamma != 0, round-half-even of 255 v;
 * both device buffers.  RT_EINVAL if a pixel has zero samples (AccumBuffer.mean). */
int rt_resolve(rt_ctx* ctx, const float* accum, int64_t npix, int32_t gamma, uint8_t* rgb);
/* ---- multi-GPU: one process, n devices of a node ------------------
 * Each device g has its own context, scene replica (identical deterministic LBVH) and
 * ZERO-initialised (H*W, 4) fp32 accumulation buffer accums[g].  split RT_SPLIT_SAMPLES:
 * device g renders global samples [s0 + g*S/n, s0 + (g+1)*S/n) (the same random numbers as
 * one GPU), then ONE grouped ncclReduce(sum, fp32) leaves the frame in accums[0];
 * RT_SPLIT_TILES: device g renders the 4-row tile bands r % n == g, and only those rows go
 * to device 0 (packed, ncclSend / ncclRecv, unpacked: the band gather below).  NCCL is
 * dlopen'ed (the process's libnccl.so.2).  rays_out (nullable): all devices' closest-hit
 * queries.  Replaces render_frame's worker split (integrators.py:426-473). */
#define RT_SPLIT_SAMPLES 0
#define RT_SPLIT_TILES 1
int rt_multi_render(int32_t n_gpus, rt_ctx* const* ctxs, rt_scene* const* scenes, const rt_render_params* p,
                    float* const* accums, int32_t split, uint64_t* rays_out);
/* ---- multi-GPU, one process per GPU (torch.distributed launches) --------
 * The same exchange as rt_multi_render, one rank per call: rank 0 makes a unique id
 * (rt_comm_unique_id), the launcher shares its RT_COMM_ID_BYTES bytes, every rank calls
 * rt_comm_create on its context's device.  Per frame, on the context stream:
 *   rt_comm_gather_bands  tile split: every rank's 4-row bands r % nranks == rank of its
 *                         (H*W, 4) fp32 accum go to rank 0's accum (rank 0's own bands are
 *                         already there); a collective: all ranks call it;
 *   rt_comm_reduce_accum  sample split: reduce(sum) of accum into rank 0's. */
typedef struct rt_comm rt_comm;
#define RT_COMM_ID_BYTES 128
int rt_comm_unique_id(uint8_t* id);
int rt_comm_create(rt_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id, rt_comm** out);
void rt_comm_destroy(rt_comm* comm);
int rt_comm_gather_bands(rt_comm* comm, rt_ctx* ctx, float* accum, int32_t width, int32_t height);
int rt_comm_reduce_accum(rt_comm* comm, rt_ctx* ctx, float* accum, int64_t npix);
/* the band gather's pack (unpack = 0: compact <- rank g's rows of accum) / unpack (accum
 * rows <- compact) on one device, without NCCL (tests); rows_out: rank g's row count */
int rt_bands_copy(rt_ctx* ctx, float* accum, float* compact, int32_t width, int32_t height, int32_t g, int32_t G,
                  int32_t unpack, int64_t* rows_out);
/* the first n raw PCG32 outputs of the (seed, pixel, sample) stream the kernels draw from
 * (sampling.py:38-79 _stream_for / _pcg_next; known-answer tests) */
int rt_stream_draws(rt_ctx* ctx, uint64_t seed, uint64_t pixel, uint64_t sample, int32_t n, uint32_t* out);
/* primary rays of sample s for every pixel of the frame (parity tests): (W*H, 8) like rt_trace_closest */
int rt_raygen(rt_ctx* ctx, const rt_render_params* p, int32_t sample, float* rays);

/* ---- two-level structure (replaces Blas / Instance / Tlas, accel.py:211-283, 339-346,
 *      439-549, and their traversal kernels accel.py:575-699, 762-895) ---------------
 * A BLAS is an rt_scene over one mesh in LOCAL space (rt_scene_create with the mesh's
 * local vertices, ids = prim, full masks) plus its float64 local normals; a custom-
 * primitive BLAS is an rt_scene over the primitives' local AABBs given as (lo, hi, lo)
 * rows, marked with rt_scene_set_custom (Blas.from_aabbs).  Both need rt_bvh_build. */
/* (n, 3) float64 local triangle normals in the reference's order (geometry.py:229-237, 274-275) */
int rt_scene_set_local_normals(rt_ctx* ctx, rt_scene* blas, const double* normals);
/* a triangle BLAS's float64 local vertices, (n, 9) in prim order (optional): with them the
 * host two-level query recomputes each hit's (t, u, v) with the reference's own float64
 * arithmetic (local ray from the float64 inverse, then _tri_hit) */
int rt_scene_set_local_rows(rt_ctx* ctx, rt_scene* blas, const double* rows);
/* custom-primitive BLAS: geometry type and the offset of its first row in the registry data */
int rt_scene_set_custom(rt_ctx* ctx, rt_scene* blas, int32_t geom_type, int64_t data_offset);
/* TLAS over n_inst instances: inst_blas[i] = the instance's BLAS, inv12 (n, 12) float64
 * instance inverses (invert_affine, accel.py:328-336), boxes6 (n, 6) fp32 world AABBs
 * (lo, hi) of the BLAS root box corners through the instance matrix (accel.py:459-469,
 * rounded outward), masks (n).  Builds the top-level LBVH.  BLAS handles are borrowed. */
int rt_tlas_create(rt_ctx* ctx, int32_t n_inst, rt_scene* const* inst_blas, const double* inv12,
                   const float* boxes6, const uint32_t* masks, rt_tlas** out);
/* Tlas.refresh_instance_bounds (accel.py:477-497): new inverses / world boxes, rebuilt
 * top level; also picks up BLASes rebuilt after a refit */
int rt_tlas_update(rt_ctx* ctx, rt_tlas* tlas, const double* inv12, const float* boxes6);
/* registry data of one custom geometry type (IntersectorRegistry, accel.py:366-392):
 * rows (n_rows, 4) float64 = sphere (cx, cy, cz, r); n_rows = 0 unregisters (a ray that
 * then reaches such a primitive fails with RT_EUNSUPPORTED) */
int rt_tlas_set_custom_data(rt_ctx* ctx, rt_tlas* tlas, int32_t geom_type, int64_t n_rows, const double* rows4);
int rt_tlas_info(rt_ctx* ctx, rt_tlas* tlas, float* root6, int32_t* height);
/* Flatten on the device into a single-level scene for rendering (the flat LBVH path of
 * rt_render): triangle instances are transformed by a kernel (float64, the host
 * flatten's order; reference-style normals from the BLAS float64 local normals), in
 * (instance, prim) order, so every triangle instance must precede the custom ones; the
 * n_custom custom primitives (spheres) are appended from host rows: world boxes as
 * (lo, hi, lo) (n_custom, 9) fp32, rt_scene_set_spheres rows, instance and prim ids.
 * mat12 (n_inst, 12) float64 instance matrices; inst_material (n_inst).  *io == NULL
 * creates the scene; otherwise a scene of the same size is refilled and rebuilt. */
int rt_tlas_flatten(rt_ctx* ctx, rt_tlas* tlas, const double* mat12, const int32_t* inst_material,
                    const float* mat_color, const float* mat_emissive, int32_t n_mat, int32_t n_custom,
                    const float* custom_boxes9, const double* custom_rows16, const int32_t* custom_inst,
                    const int32_t* custom_prim, int32_t bits, rt_scene** io);
void rt_tlas_destroy(rt_tlas* tlas);
/* closest_hit_batch / any_hit_batch over the two-level structure, host float64 rays,
 * outputs and conventions as rt_closest_hit_host / rt_any_hit_host (inst = instance
 * index, prim = primitive index in its BLAS) */
int rt_tlas_closest_host(rt_ctx* ctx, rt_tlas* tlas, int64_t n, const double* origins, const double* dirs,
                         const double* t_min, const double* t_max, double t_min_s, double t_max_s,
                         uint32_t ray_mask, double* t, int64_t* inst, int64_t* prim, double* u, double* v,
                         double* normal, int64_t* stats);
int rt_tlas_any_host(rt_ctx* ctx, rt_tlas* tlas, int64_t n, const double* origins, const double* dirs,
                     const double* t_min, const double* t_max, double t_min_s, double t_max_s,
                     uint32_t ray_mask, uint8_t* hit);

#ifdef __cplusplus
}
#endif
#endif
