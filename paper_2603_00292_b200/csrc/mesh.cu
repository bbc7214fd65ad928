// mesh.cu -- indexed meshes on the device: compile_scene's geometry side (scene.py:79-141,
// Blas.from_mesh accel.py:223-236) and Blas.refit (accel.py:263-283).
//
// rt_mesh_upload  one H2D of the reference's own float64 vertices / int64 faces, validated
//                 on the device (the BuildError checks of Blas.from_mesh) with the mesh's
//                 float64 root box reduced in the same pass;
// rt_scene_compile  every instance of every mesh written into the flat scene by one kernel
//                 per mesh: world fp32 rows, reference-order float64 world normals, the
//                 float64 local rows of the host query, ids / masks / materials;
// rt_scene_refit_mesh  new vertices for a resident mesh, same kernel.
#include <limits.h>
#include <math.h>
#include <string.h>

#include <vector>

#include "rt_common.cuh"
struct rt_mesh {
    int device;
    cudaStream_t stream;  // storage: stream-ordered pool memory freed on this stream
    int64_t nv, nf;
    int32_t n_inst;
    int32_t local;        // RT_MESH_LOCAL: rows = the local vertices, float64 local normals
    int3* faces;          // (nf) device
    double* xform;        // (n_inst, 21) device
    int64_t* offset;      // (n_inst) device: first flat triangle of each instance
    double* verts;        // (nv, 3) device: the latest uploaded vertices (float64, or fp32 for an fp32 refit)
    int4* meta;           // (n_inst) device, compiled scenes: (instance id, material, mask, 0) per placement
    int64_t bounds_nv;    // rt_mesh_upload: vertices referenced by faces have float64 bounds `bounds`
    double bounds[6];
    unsigned long long* d_red;  // (8) device: bounds re-reduced by each refit (orderable encoding)
    int bounds_dirty;           // d_red is newer than `bounds`
    int pending;                // rt_mesh_upload_async: validation not read back yet
};

namespace {

// world triangles + world normals of every (instance, face): scene.py compile_scene's
// float64 expressions in their evaluation order, each operation correctly rounded
// (__dmul_rn / __dadd_rn / __dsub_rn keep nvcc from contracting them into FMAs)
__device__ __forceinline__ double dot3_affine(const double* m, double x, double y, double z) {
    return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[0], x), __dmul_rn(m[1], y)), __dmul_rn(m[2], z)), m[3]);
}

template <typename T>
__global__ void refit_mesh_kernel(int64_t nf, int32_t n_inst, const int3* __restrict__ faces,
                                  const T* __restrict__ Vt, const double* __restrict__ xform,
                                  const int64_t* __restrict__ offset, float* __restrict__ tris,
                                  float4* __restrict__ attr, double* __restrict__ lnormal64,
                                  double* __restrict__ lrows64, double* __restrict__ wnormal64,
                                  const int4* __restrict__ meta, int32_t* __restrict__ tri_inst,
                                  int32_t* __restrict__ tri_prim, uint32_t* __restrict__ tri_mask,
                                  const unsigned long long* __restrict__ verdict) {
    // a compile enqueued behind its mesh's validation (rt_mesh_upload_async) writes nothing
    // for a mesh that failed it (its narrowed faces may point anywhere)
    if (verdict && (verdict[6] != ULLONG_MAX || verdict[7] != ULLONG_MAX)) return;
    const int64_t total = nf * n_inst;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = (int32_t)(q / nf);
        const int64_t k = q - (int64_t)j * nf;
        const double* m = xform + 21 * j;
        const double* inv = m + 12;
        const int3 f = faces[k];
        // fp32 vertices widen exactly: the same float64 values compile_scene would see
        const double a[3] = {(double)Vt[3 * (int64_t)f.x], (double)Vt[3 * (int64_t)f.x + 1], (double)Vt[3 * (int64_t)f.x + 2]};
        const double b[3] = {(double)Vt[3 * (int64_t)f.y], (double)Vt[3 * (int64_t)f.y + 1], (double)Vt[3 * (int64_t)f.y + 2]};
        const double c[3] = {(double)Vt[3 * (int64_t)f.z], (double)Vt[3 * (int64_t)f.z + 1], (double)Vt[3 * (int64_t)f.z + 2]};
        float* t = tris + 9 * (offset[j] + k);
        const double* vs[3] = {a, b, c};
        double* rows64 = lrows64 ? lrows64 + 9 * (offset[j] + k) : nullptr;
        if (rows64 && !lnormal64) {   // a flat scene keeping its local vertices for the query
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int r = 0; r < 3; ++r) rows64[3 * v + r] = vs[v][r];
        }
        if (lnormal64) {       // a BLAS: its rows are the local vertices themselves (Blas._rows)
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    t[3 * v + r] = __double2float_rn(vs[v][r]);
                    if (rows64) rows64[3 * v + r] = vs[v][r];
                }
        } else {
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int r = 0; r < 3; ++r)
                    t[3 * v + r] = __double2float_rn(dot3_affine(m + 4 * r, vs[v][0], vs[v][1], vs[v][2]));
        }
        // local normal (geometry.py:229-237): e0 = b - a, e1 = c - b, n = e0 x e1 / |n|
        const double e0x = __dsub_rn(b[0], a[0]), e0y = __dsub_rn(b[1], a[1]), e0z = __dsub_rn(b[2], a[2]);
        const double e1x = __dsub_rn(c[0], b[0]), e1y = __dsub_rn(c[1], b[1]), e1z = __dsub_rn(c[2], b[2]);
        const double nx = __dsub_rn(__dmul_rn(e0y, e1z), __dmul_rn(e0z, e1y));
        const double ny = __dsub_rn(__dmul_rn(e0z, e1x), __dmul_rn(e0x, e1z));
        const double nz = __dsub_rn(__dmul_rn(e0x, e1y), __dmul_rn(e0y, e1x));
        const double nlen = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny)), __dmul_rn(nz, nz)));
        const double lx = __ddiv_rn(nx, nlen), ly = __ddiv_rn(ny, nlen), lz = __ddiv_rn(nz, nlen);
        if (lnormal64) {       // the two-level kernels transform the float64 local normal per hit
            double* ln = lnormal64 + 3 * (offset[j] + k);
            ln[0] = lx; ln[1] = ly; ln[2] = lz;
            continue;
        }
        // world normal (accel.py:843-847): inverse-transpose sum, times 1 / sqrt(|w|^2)
        const double wx = __dadd_rn(__dadd_rn(__dmul_rn(inv[0], lx), __dmul_rn(inv[3], ly)), __dmul_rn(inv[6], lz));
        const double wy = __dadd_rn(__dadd_rn(__dmul_rn(inv[1], lx), __dmul_rn(inv[4], ly)), __dmul_rn(inv[7], lz));
        const double wz = __dadd_rn(__dadd_rn(__dmul_rn(inv[2], lx), __dmul_rn(inv[5], ly)), __dmul_rn(inv[8], lz));
        const double il =
            __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)), __dmul_rn(wz, wz))));
        const double nwx = __dmul_rn(wx, il), nwy = __dmul_rn(wy, il), nwz = __dmul_rn(wz, il);
        float4* at = attr + offset[j] + k;
        float w;
        if (meta) {                                     // compile: ids, mask and material of the placement
            const int4 mt = meta[j];
            tri_inst[offset[j] + k] = mt.x;
            tri_prim[offset[j] + k] = (int32_t)k;
            tri_mask[offset[j] + k] = (uint32_t)mt.z;
            w = __int_as_float(mt.y);
        } else {
            w = at->w;                                  // refit: material index bits stay
        }
        *at = make_float4(__double2float_rn(nwx), __double2float_rn(nwy), __double2float_rn(nwz), w);
        if (wnormal64) {
            double* wn = wnormal64 + 3 * (offset[j] + k);
            wn[0] = nwx; wn[1] = nwy; wn[2] = nwz;
        }
    }
}

// normals of world triangles given directly (GpuTlas.refit): the same float64 expressions
// with an identity instance frame (its inverse-transpose sum is exact, the renormalisation
// is kept)
__global__ void normals_from_tris_kernel(int64_t n, const float* __restrict__ tris, float4* __restrict__ attr,
                                         double* __restrict__ wnormal64) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float* t = tris + 9 * i;
        const double e0x = __dsub_rn(t[3], t[0]), e0y = __dsub_rn(t[4], t[1]), e0z = __dsub_rn(t[5], t[2]);
        const double e1x = __dsub_rn(t[6], t[3]), e1y = __dsub_rn(t[7], t[4]), e1z = __dsub_rn(t[8], t[5]);
        const double nx = __dsub_rn(__dmul_rn(e0y, e1z), __dmul_rn(e0z, e1y));
        const double ny = __dsub_rn(__dmul_rn(e0z, e1x), __dmul_rn(e0x, e1z));
        const double nz = __dsub_rn(__dmul_rn(e0x, e1y), __dmul_rn(e0y, e1x));
        const double nlen = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny)), __dmul_rn(nz, nz)));
        const double lx = __ddiv_rn(nx, nlen), ly = __ddiv_rn(ny, nlen), lz = __ddiv_rn(nz, nlen);
        const double il =
            __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(lx, lx), __dmul_rn(ly, ly)), __dmul_rn(lz, lz))));
        const double wx = __dmul_rn(lx, il), wy = __dmul_rn(ly, il), wz = __dmul_rn(lz, il);
        float4 a = attr[i];
        a.x = __double2float_rn(wx);
        a.y = __double2float_rn(wy);
        a.z = __double2float_rn(wz);
        attr[i] = a;
        if (wnormal64) { wnormal64[3 * i] = wx; wnormal64[3 * i + 1] = wy; wnormal64[3 * i + 2] = wz; }
    }
}

}  // namespace

extern "C" {

int rt_scene_update_normals(rt_ctx* c, rt_scene* s) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    // new world rows: the local vertices / frames no longer describe them
    if (s->inst_inv64) {
        RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
        rt_free(s->inst_inv64, s->stream);
        s->inst_inv64 = nullptr;
    }
    const int64_t n = s->n - s->n_spheres;
    if (n <= 0) return RT_OK;
    int64_t grid = (n + 255) / 256;
    if (grid > (int64_t)c->num_sms * 16) grid = (int64_t)c->num_sms * 16;
    normals_from_tris_kernel<<<(unsigned)grid, 256, 0, c->stream>>>(n, s->tris, s->tri_attr, s->wnormal64);
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

int rt_scene_set_local_frames(rt_ctx* c, rt_scene* s, int32_t n_inst, const double* inv12, const double* rows9) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && n_inst >= 1 && inv12 && rows9, "NULL argument or no instance");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_free(s->inst_inv64, s->stream);
    s->inst_inv64 = nullptr;
    RT_CUDA_TRY(rt_alloc((void**)&s->inst_inv64, sizeof(double) * 12 * (size_t)n_inst, s->stream));
    RT_CUDA_TRY(cudaMemcpy(s->inst_inv64, inv12, sizeof(double) * 12 * (size_t)n_inst, cudaMemcpyHostToDevice));
    if (!s->lrows64) RT_CUDA_TRY(rt_alloc((void**)&s->lrows64, sizeof(double) * 9 * (size_t)s->n, s->stream));
    RT_CUDA_TRY(cudaMemcpy(s->lrows64, rows9, sizeof(double) * 9 * (size_t)s->n, cudaMemcpyHostToDevice));
    return RT_OK;
}

int rt_scene_set_normals64(rt_ctx* c, rt_scene* s, const double* n3) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && n3, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    if (!s->wnormal64) RT_CUDA_TRY(rt_alloc((void**)&s->wnormal64, sizeof(double) * 3 * (size_t)s->n, s->stream));
    RT_CUDA_TRY(cudaMemcpy(s->wnormal64, n3, sizeof(double) * 3 * (size_t)s->n, cudaMemcpyHostToDevice));
    return RT_OK;
}

int rt_scene_get_vertices(rt_ctx* c, rt_scene* s, float* tris) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && tris, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_CUDA_TRY(cudaMemcpyAsync(tris, s->tris, sizeof(float) * 9 * s->n, cudaMemcpyDeviceToHost, c->stream));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return RT_OK;
}

int rt_mesh_create(rt_ctx* c, int64_t n_vertices, int64_t n_faces, const int32_t* faces, int32_t n_inst,
                   const double* xform, const int64_t* tri_offset, int32_t flags, rt_mesh** out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && faces && xform && tri_offset && out, "NULL argument");
    RT_CHECK_ARG(n_vertices >= 3 && n_faces >= 1 && n_inst >= 1, "empty mesh or no instance");
    RT_CHECK_ARG(!(flags & RT_MESH_LOCAL) || n_inst == 1, "a local (BLAS) mesh has exactly one placement");
    for (int64_t k = 0; k < 3 * n_faces; ++k)
        RT_CHECK_ARG(faces[k] >= 0 && faces[k] < n_vertices, "face index out of range");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_mesh* m = new rt_mesh();
    m->device = c->device;
    m->nv = n_vertices;
    m->nf = n_faces;
    m->n_inst = n_inst;
    m->local = (flags & RT_MESH_LOCAL) ? 1 : 0;
    m->stream = c->stream;
    cudaError_t e = rt_alloc((void**)&m->faces, sizeof(int3) * n_faces, c->stream, false);
    if (e == cudaSuccess) e = rt_alloc((void**)&m->xform, sizeof(double) * 21 * n_inst, c->stream, false);
    if (e == cudaSuccess) e = rt_alloc((void**)&m->offset, sizeof(int64_t) * n_inst, c->stream, false);
    if (e == cudaSuccess) e = rt_alloc((void**)&m->verts, sizeof(double) * 3 * n_vertices, c->stream);
    if (e == cudaSuccess) e = cudaMemcpy(m->faces, faces, sizeof(int3) * n_faces, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(m->xform, xform, sizeof(double) * 21 * n_inst, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(m->offset, tri_offset, sizeof(int64_t) * n_inst, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        rt_mesh_destroy(m);
        rt_set_error("rt_mesh_create: %s", cudaGetErrorString(e));
        return RT_ECUDA;
    }
    *out = m;
    return RT_OK;
}

}  // extern "C"

namespace {

// one launch of the placement kernel over every (instance, face) of mesh m
int launch_mesh(rt_ctx* c, rt_scene* s, rt_mesh* m, bool f32, bool with_meta) {
    double* ln = m->local ? s->lnormal64 : nullptr;
    const int64_t total = m->nf * m->n_inst;
    if (total == 0) return RT_OK;
    int64_t grid = (total + 255) / 256;
    if (grid > (int64_t)c->num_sms * 16) grid = (int64_t)c->num_sms * 16;
    const int4* meta = with_meta ? m->meta : nullptr;
    const unsigned long long* verdict = m->pending ? m->d_red : nullptr;
    double* wn = m->local ? nullptr : s->wnormal64;
    if (f32)
        refit_mesh_kernel<float><<<(unsigned)grid, 256, 0, c->stream>>>(
            m->nf, m->n_inst, m->faces, reinterpret_cast<const float*>(m->verts), m->xform, m->offset, s->tris,
            s->tri_attr, ln, s->lrows64, wn, meta, s->tri_inst, s->tri_prim, s->tri_mask, verdict);
    else
        refit_mesh_kernel<double><<<(unsigned)grid, 256, 0, c->stream>>>(
            m->nf, m->n_inst, m->faces, m->verts, m->xform, m->offset, s->tris, s->tri_attr, ln, s->lrows64, wn,
            meta, s->tri_inst, s->tri_prim, s->tri_mask, verdict);
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

// orderable uint64 encoding of float64 (atomicMin / atomicMax of the mesh bounds)
__device__ __forceinline__ unsigned long long d2ord(double d) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u >> 63) ? ~u : (u | (1ull << 63));
}
__host__ __device__ __forceinline__ double ord2d(unsigned long long u) {
    u = (u >> 63) ? (u & ~(1ull << 63)) : ~u;
    double d;
    memcpy(&d, &u, 8);
    return d;
}

// Blas.from_mesh's checks (accel.py:223-236) for one mesh in one pass: the int64 faces
// are range-checked and narrowed to int3, each triangle's 9 coordinates are checked
// for non-finite values (== ~isfinite(lo|hi) of _triangle_boxes), and the float64 root
// box (the union of the triangle boxes) is reduced.  red: [0..2] min, [3..5] max
// (orderable), [6] first face with an out-of-range index, [7] first non-finite triangle.
__global__ void mesh_check_kernel(int64_t nf, int64_t nv, const int64_t* __restrict__ F,
                                  const double* __restrict__ V, int3* __restrict__ F32,
                                  unsigned long long* __restrict__ red) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    unsigned long long bad_face = ULLONG_MAX, bad_prim = ULLONG_MAX;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = F[3 * k], i1 = F[3 * k + 1], i2 = F[3 * k + 2];
        if (i0 < 0 || i0 >= nv || i1 < 0 || i1 >= nv || i2 < 0 || i2 >= nv) {
            bad_face = min(bad_face, (unsigned long long)k);
            F32[k] = make_int3(0, 0, 0);
            continue;
        }
        F32[k] = make_int3((int)i0, (int)i1, (int)i2);
        const int64_t id[3] = {i0, i1, i2};
        double x[9];
        bool fin = true;
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                x[3 * v + r] = V[3 * id[v] + r];
                fin = fin && isfinite(x[3 * v + r]);
            }
        if (!fin) {
            bad_prim = min(bad_prim, (unsigned long long)k);
            continue;
        }
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                lo[r] = fmin(lo[r], x[3 * v + r]);
                hi[r] = fmax(hi[r], x[3 * v + r]);
            }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            lo[r] = fmin(lo[r], __shfl_xor_sync(0xFFFFFFFFu, lo[r], o));
            hi[r] = fmax(hi[r], __shfl_xor_sync(0xFFFFFFFFu, hi[r], o));
        }
        bad_face = min(bad_face, __shfl_xor_sync(0xFFFFFFFFu, bad_face, o));
        bad_prim = min(bad_prim, __shfl_xor_sync(0xFFFFFFFFu, bad_prim, o));
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            if (lo[r] <= hi[r]) {
                atomicMin(red + r, d2ord(lo[r]));
                atomicMax(red + 3 + r, d2ord(hi[r]));
            }
        }
        if (bad_face != ULLONG_MAX) atomicMin(red + 6, bad_face);
        if (bad_prim != ULLONG_MAX) atomicMin(red + 7, bad_prim);
    }
}

// the float64 root box of a resident mesh's current vertices (after a refit): the union of
// its triangle boxes, as _triangle_boxes + _refit_boxes give the reference's root bounds
template <typename T>
__global__ void mesh_bounds_kernel(int64_t nf, const int3* __restrict__ F, const T* __restrict__ V,
                                   unsigned long long* __restrict__ red) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf; k += (int64_t)gridDim.x * blockDim.x) {
        const int3 f = F[k];
        const int64_t id[3] = {f.x, f.y, f.z};
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const double x = (double)V[3 * id[v] + r];
                lo[r] = fmin(lo[r], x);
                hi[r] = fmax(hi[r], x);
            }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            lo[r] = fmin(lo[r], __shfl_xor_sync(0xFFFFFFFFu, lo[r], o));
            hi[r] = fmax(hi[r], __shfl_xor_sync(0xFFFFFFFFu, hi[r], o));
        }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int r = 0; r < 3; ++r)
            if (lo[r] <= hi[r]) {
                atomicMin(red + r, d2ord(lo[r]));
                atomicMax(red + 3 + r, d2ord(hi[r]));
            }
}

__global__ void red_init_kernel(unsigned long long* red) {
    if (threadIdx.x < 8) red[threadIdx.x] = (threadIdx.x < 3 || threadIdx.x >= 6) ? ULLONG_MAX : 0ull;
}

// ids / rows of the custom primitives (sphere instances) at the end of the flat scene
struct CustomRow {
    float box[9];
    int32_t material;
    uint32_t mask;
};

}  // namespace

extern "C" {

int rt_scene_refit_mesh(rt_ctx* c, rt_scene* s, rt_mesh* m, int64_t n_vertices, const void* vertices,
                        int32_t vertices_f32) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s && m && vertices, "NULL argument");
    RT_CHECK_ARG(m->device == c->device, "mesh and context live on different devices");
    RT_CHECK_ARG(m->n_inst >= 1 && m->xform, "mesh has no placement in a scene");
    if (n_vertices != m->nv) {
        rt_set_error("vertex count changed (%lld -> %lld)", (long long)m->nv, (long long)n_vertices);
        return RT_EINVAL;
    }
    if (m->local && !s->lnormal64) {
        rt_set_error("a local (BLAS) mesh refits a scene with float64 local normals");
        return RT_EINVAL;
    }
    RT_CUDA_TRY(cudaSetDevice(c->device));
    const size_t vbytes = (vertices_f32 ? sizeof(float) : sizeof(double)) * 3 * m->nv;
    int rc = rt_h2d(c, m->verts, vertices, vbytes);
    if (rc) return rc;
    rc = launch_mesh(c, s, m, vertices_f32 != 0, false);
    if (rc) return rc;
    if (m->d_red) {       // the mesh's new root box (read back only when asked, rt_mesh_info)
        red_init_kernel<<<1, 32, 0, c->stream>>>(m->d_red);
        int64_t grid = (m->nf + 255) / 256;
        if (grid > (int64_t)c->num_sms * 4) grid = (int64_t)c->num_sms * 4;
        if (vertices_f32)
            mesh_bounds_kernel<float><<<(unsigned)grid, 256, 0, c->stream>>>(
                m->nf, m->faces, reinterpret_cast<const float*>(m->verts), m->d_red);
        else
            mesh_bounds_kernel<double><<<(unsigned)grid, 256, 0, c->stream>>>(m->nf, m->faces, m->verts, m->d_red);
        RT_CUDA_TRY(cudaGetLastError());
        m->bounds_dirty = 1;
    }
    s->built = 0;
    return RT_OK;
}

}  // extern "C"

// rt_mesh_upload's two halves: the copies, the validation kernel and the root-box reduction
// enqueued on the context stream; then one small read-back and the verdict.  Between them
// the host is free (rt_mesh_upload_async / rt_mesh_upload_finish): compile_scene prepares
// its instance tables while the mesh crosses PCIe.
// rt_scene_compile's small host tables (materials, instance frames, offsets, ids) go up
// from one pinned staging buffer: an async copy from pageable memory waits for the copy
// engine to drain (here: the meshes' own uploads still in flight), a pinned one is queued
struct TableStage {
    struct Item { void* dst; size_t off, bytes; };
    std::vector<char> host;
    std::vector<Item> items;
    void add(void* dst, const void* src, size_t bytes) {
        const size_t off = (host.size() + 255) & ~(size_t)255;
        host.resize(off + bytes);
        memcpy(host.data() + off, src, bytes);
        items.push_back({dst, off, bytes});
    }
    cudaError_t flush(rt_ctx* c) {
        if (host.empty()) return cudaSuccess;
        cudaError_t e = cudaSuccess;
        if (!c->tab_ev) {
            e = cudaEventCreateWithFlags(&c->tab_ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        if (c->h_tab_bytes < host.size()) {
            if (c->h_tab) {
                cudaEventSynchronize(c->tab_ev);
                cudaFreeHost(c->h_tab);
                c->h_tab = nullptr;
                c->h_tab_bytes = 0;
            }
            size_t cap = 64 << 10;
            while (cap < host.size()) cap *= 2;
            e = cudaHostAlloc(&c->h_tab, cap, cudaHostAllocDefault);
            if (e != cudaSuccess) return e;
            c->h_tab_bytes = cap;
        } else {
            e = cudaEventSynchronize(c->tab_ev);   // the previous compile's copies are done
            if (e != cudaSuccess) return e;
        }
        memcpy(c->h_tab, host.data(), host.size());
        for (const Item& it : items) {
            e = cudaMemcpyAsync(it.dst, static_cast<char*>(c->h_tab) + it.off, it.bytes, cudaMemcpyHostToDevice,
                                c->stream);
            if (e != cudaSuccess) return e;
        }
        return cudaEventRecord(c->tab_ev, c->stream);
    }
};

static int mesh_upload_enqueue(rt_ctx* c, int64_t n_vertices, const double* vertices, int64_t n_faces,
                               const int64_t* faces, rt_mesh** out) {
    RT_CHECK_ARG(c && out, "NULL argument");
    RT_CHECK_ARG(n_vertices >= 0 && n_faces >= 0 && (n_vertices == 0 || vertices) && (n_faces == 0 || faces),
                 "bad mesh arrays");
    if (n_faces == 0) {
        rt_set_error("cannot build over zero primitives");
        return RT_EBUILD;
    }
    RT_CHECK_ARG(n_vertices < (1ll << 31) && n_faces < (1ll << 30), "mesh too large (2^31 vertices, 2^30 faces)");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_mesh* m = new rt_mesh();
    memset(m, 0, sizeof *m);
    m->device = c->device;
    m->nv = n_vertices;
    m->nf = n_faces;
    cudaStream_t st = c->stream;
    m->stream = st;
    int64_t* f64 = nullptr;
    unsigned long long* red = nullptr;
    cudaError_t e = rt_alloc((void**)&m->faces, sizeof(int3) * n_faces, st, false);
    if (e == cudaSuccess) e = rt_alloc((void**)&m->verts, sizeof(double) * 3 * (n_vertices > 0 ? n_vertices : 1), st, false);
    if (e == cudaSuccess) e = cudaMallocAsync(&f64, sizeof(int64_t) * 3 * n_faces, st);
    if (e == cudaSuccess) e = rt_alloc((void**)&red, sizeof(unsigned long long) * 8, st, false);
    if (e == cudaSuccess && n_vertices > 0 && rt_h2d(c, m->verts, vertices, sizeof(double) * 3 * n_vertices))
        e = cudaErrorUnknown;
    if (e == cudaSuccess && rt_h2d(c, f64, faces, sizeof(int64_t) * 3 * n_faces)) e = cudaErrorUnknown;
    if (e == cudaSuccess) {
        red_init_kernel<<<1, 32, 0, st>>>(red);
        int64_t grid = (n_faces + 255) / 256;
        if (grid > (int64_t)c->num_sms * 8) grid = (int64_t)c->num_sms * 8;
        mesh_check_kernel<<<(unsigned)grid, 256, 0, st>>>(n_faces, n_vertices, f64, m->verts, m->faces, red);
        e = cudaGetLastError();
    }
    if (f64) cudaFreeAsync(f64, st);
    m->d_red = red;       // kept: each refit re-reduces the bounds into it
    if (e != cudaSuccess) {
        cudaStreamSynchronize(st);
        rt_mesh_destroy(m);
        rt_set_error("rt_mesh_upload: %s", cudaGetErrorString(e));
        return RT_ECUDA;
    }
    m->pending = 1;
    *out = m;
    return RT_OK;
}

static int mesh_upload_finish(rt_mesh* m, double* bounds6) {
    RT_CHECK_ARG(m, "mesh is NULL");
    if (!m->pending) {
        if (bounds6) memcpy(bounds6, m->bounds, sizeof m->bounds);
        if (m->bounds_nv == m->nv) return RT_OK;
        rt_set_error("mesh was not uploaded by rt_mesh_upload_async");
        return RT_ESTATE;
    }
    RT_CUDA_TRY(cudaSetDevice(m->device));
    unsigned long long r[8];
    cudaError_t e = cudaMemcpyAsync(r, m->d_red, sizeof r, cudaMemcpyDeviceToHost, m->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(m->stream);
    if (e != cudaSuccess) {
        rt_set_error("rt_mesh_upload: %s", cudaGetErrorString(e));
        return RT_ECUDA;
    }
    m->pending = 0;
    if (r[6] != ULLONG_MAX) {
        rt_set_error("face index out of range");
        return RT_EBUILD;
    }
    if (r[7] != ULLONG_MAX) {
        rt_set_error("non-finite bounds for primitive %llu", r[7]);
        return RT_EBUILD;
    }
    for (int k = 0; k < 6; ++k) m->bounds[k] = ord2d(r[k]);
    m->bounds_nv = m->nv;
    if (bounds6) memcpy(bounds6, m->bounds, sizeof m->bounds);
    return RT_OK;
}

extern "C" {

int rt_mesh_upload(rt_ctx* c, int64_t n_vertices, const double* vertices, int64_t n_faces, const int64_t* faces,
                   double* bounds6, rt_mesh** out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && out && bounds6, "NULL argument");
    rt_mesh* m = nullptr;
    int rc = mesh_upload_enqueue(c, n_vertices, vertices, n_faces, faces, &m);
    if (rc) return rc;
    rc = mesh_upload_finish(m, bounds6);
    if (rc) {
        rt_mesh_destroy(m);
        return rc;
    }
    *out = m;
    return RT_OK;
}

int rt_mesh_upload_async(rt_ctx* c, int64_t n_vertices, const double* vertices, int64_t n_faces,
                         const int64_t* faces, rt_mesh** out) {
    RT_CTX_LOCK(c);
    return mesh_upload_enqueue(c, n_vertices, vertices, n_faces, faces, out);
}

int rt_mesh_upload_finish(rt_ctx* c, rt_mesh* m, double* bounds6) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && m, "NULL argument");
    RT_CHECK_ARG(m->device == c->device, "mesh and context live on different devices");
    return mesh_upload_finish(m, bounds6);
}

int rt_scene_compile(rt_ctx* c, int32_t n_meshes, rt_mesh* const* meshes, int32_t n_inst,
                     const rt_instance_src* inst, int32_t n_custom, const rt_custom_src* custom,
                     const float* mat_color, const float* mat_emissive, int32_t n_mat, rt_scene** out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && out, "NULL argument");
    RT_CHECK_ARG(n_meshes >= 0 && n_inst >= 0 && n_custom >= 0, "negative count");
    RT_CHECK_ARG(n_inst + n_custom >= 1, "a scene needs at least one instance");
    RT_CHECK_ARG((n_inst == 0 || (inst && meshes)) && (n_custom == 0 || custom), "NULL instance table");
    RT_CHECK_ARG(n_mat >= 1 && mat_color && mat_emissive, "materials missing");
    int64_t n = n_custom;
    for (int32_t i = 0; i < n_inst; ++i) {
        const rt_instance_src& d = inst[i];
        if (d.mesh < 0 || d.mesh >= n_meshes || !meshes[d.mesh]) {
            rt_set_error("instance %d references unknown mesh %d", i, d.mesh);
            return RT_EINVAL;
        }
        if (!meshes[d.mesh]->pending && meshes[d.mesh]->bounds_nv != meshes[d.mesh]->nv && !meshes[d.mesh]->local) {
            rt_set_error("instance %d: mesh %d failed its validation", i, d.mesh);
            return RT_ESTATE;
        }
        if (meshes[d.mesh]->device != c->device || meshes[d.mesh]->local) {
            rt_set_error("instance %d: mesh lives on another device or is a BLAS mesh", i);
            return RT_EINVAL;
        }
        if (d.material < 0 || d.material >= n_mat) {
            rt_set_error("instance %d references material %d of %d", i, d.material, n_mat);
            return RT_EINVAL;
        }
        n += meshes[d.mesh]->nf;
    }
    for (int32_t k = 0; k < n_custom; ++k) {
        if (custom[k].material < 0 || custom[k].material >= n_mat) {
            rt_set_error("custom primitive %d references material %d of %d", k, custom[k].material, n_mat);
            return RT_EINVAL;
        }
        RT_CHECK_ARG(custom[k].row[15] > 0.0, "sphere radius must be > 0");
    }
    RT_CUDA_TRY(cudaSetDevice(c->device));
    rt_scene* s = nullptr;
    bool pending = false;                         // validation still in flight: rt_mesh_upload_finish syncs
    for (int32_t k = 0; k < n_meshes; ++k) pending |= meshes[k] && meshes[k]->pending;
    int rc = rt_scene_alloc_ex(c, n, n_mat, &s, pending ? 0 : 1);
    if (rc) return rc;
    auto fail = [&](int code) {
        rt_scene_destroy(s);
        return code;
    };
    TableStage tab;
    {
        std::vector<float4> mc(n_mat), me(n_mat);
        for (int k = 0; k < n_mat; ++k) {
            mc[k] = make_float4(mat_color[3 * k], mat_color[3 * k + 1], mat_color[3 * k + 2], 0.f);
            me[k] = make_float4(mat_emissive[3 * k], mat_emissive[3 * k + 1], mat_emissive[3 * k + 2], 0.f);
        }
        tab.add(s->mat_color, mc.data(), sizeof(float4) * n_mat);
        tab.add(s->mat_emissive, me.data(), sizeof(float4) * n_mat);
    }
    cudaStream_t st = c->stream;
    cudaError_t e = rt_alloc((void**)&s->wnormal64, sizeof(double) * 3 * (size_t)n, st, false);
    if (e == cudaSuccess) e = rt_alloc((void**)&s->lrows64, sizeof(double) * 9 * (size_t)n, st, false);
    const int32_t ni = n_inst + n_custom;
    if (e == cudaSuccess) e = rt_alloc((void**)&s->inst_inv64, sizeof(double) * 12 * (size_t)ni, st, false);
    if (e != cudaSuccess) {
        rt_set_error("cudaMalloc failed: %s", cudaGetErrorString(e));
        return fail(RT_ENOMEM);
    }
    // instance inverses (the host query's local-space refinement): instances, then customs
    std::vector<double> inv(12 * (size_t)ni);
    for (int32_t i = 0; i < n_inst; ++i) memcpy(&inv[12 * (size_t)i], inst[i].inverse, 12 * sizeof(double));
    for (int32_t k = 0; k < n_custom; ++k) memcpy(&inv[12 * (size_t)(n_inst + k)], custom[k].row, 12 * sizeof(double));
    // per mesh: its placements (3x4 matrix + 3x3 inverse block, first flat id, ids)
    std::vector<std::vector<double>> xf(n_meshes);
    std::vector<std::vector<int64_t>> ofs(n_meshes);
    std::vector<std::vector<int4>> meta(n_meshes);
    int64_t off = 0;
    for (int32_t i = 0; i < n_inst; ++i) {
        const rt_instance_src& d = inst[i];
        std::vector<double>& x = xf[d.mesh];
        x.insert(x.end(), d.matrix, d.matrix + 12);
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) x.push_back(d.inverse[4 * r + q]);
        ofs[d.mesh].push_back(off);
        meta[d.mesh].push_back(make_int4(i, d.material, (int)d.mask, 0));
        off += meshes[d.mesh]->nf;
    }
    tab.add(s->inst_inv64, inv.data(), sizeof(double) * inv.size());
    for (int32_t k = 0; k < n_meshes && e == cudaSuccess; ++k) {
        rt_mesh* m = meshes[k];
        if (!m || ofs[k].empty()) continue;
        const int32_t cnt = (int32_t)ofs[k].size();
        if (m->n_inst != cnt) {
            rt_free(m->xform, m->stream);
            rt_free(m->offset, m->stream);
            rt_free(m->meta, m->stream);
            m->xform = nullptr; m->offset = nullptr; m->meta = nullptr;
            m->n_inst = 0;
            e = rt_alloc((void**)&m->xform, sizeof(double) * 21 * cnt, m->stream, false);
            if (e == cudaSuccess) e = rt_alloc((void**)&m->offset, sizeof(int64_t) * cnt, m->stream, false);
            if (e == cudaSuccess) e = rt_alloc((void**)&m->meta, sizeof(int4) * cnt, m->stream, false);
            if (e != cudaSuccess) break;
            m->n_inst = cnt;
        }
        tab.add(m->xform, xf[k].data(), sizeof(double) * 21 * cnt);
        tab.add(m->offset, ofs[k].data(), sizeof(int64_t) * cnt);
        tab.add(m->meta, meta[k].data(), sizeof(int4) * cnt);
    }
    if (e == cudaSuccess) e = tab.flush(c);       // every table, then the kernels that read them
    for (int32_t k = 0; k < n_meshes && e == cudaSuccess; ++k) {
        rt_mesh* m = meshes[k];
        if (!m || ofs[k].empty()) continue;
        rc = launch_mesh(c, s, m, false, true);
        if (rc) return fail(rc);
    }
    if (e == cudaSuccess && n_custom > 0) {
        // custom primitives after every triangle (scene.py:101-112): box rows, ids, zero normals
        const int64_t b = n - n_custom;
        std::vector<float> rows(9 * (size_t)n_custom);
        std::vector<float4> attr(n_custom);
        std::vector<int32_t> ids(n_custom), prims(n_custom, 0);
        std::vector<uint32_t> masks(n_custom);
        std::vector<double> sph(16 * (size_t)n_custom);
        for (int32_t k = 0; k < n_custom; ++k) {
            memcpy(&rows[9 * (size_t)k], custom[k].box, 9 * sizeof(float));
            float w;
            memcpy(&w, &custom[k].material, 4);
            attr[k] = make_float4(0.f, 0.f, 0.f, w);
            ids[k] = n_inst + k;
            masks[k] = custom[k].mask;
            memcpy(&sph[16 * (size_t)k], custom[k].row, 16 * sizeof(double));
        }
        e = cudaMemcpy(s->tris + 9 * b, rows.data(), sizeof(float) * rows.size(), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(s->tri_attr + b, attr.data(), sizeof(float4) * n_custom, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(s->tri_inst + b, ids.data(), 4 * (size_t)n_custom, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(s->tri_prim + b, prims.data(), 4 * (size_t)n_custom, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(s->tri_mask + b, masks.data(), 4 * (size_t)n_custom, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemsetAsync(s->wnormal64 + 3 * b, 0, sizeof(double) * 3 * n_custom, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(s->lrows64 + 9 * b, 0, sizeof(double) * 9 * n_custom, st);
        if (e == cudaSuccess) {
            rc = rt_scene_set_spheres(c, s, n_custom, sph.data());
            if (rc) return fail(rc);
        }
    }
    if (e == cudaSuccess) e = cudaGetLastError();   // (kernel faults surface at the next sync)
    // every block usable from any stream before the scene is returned -- or, with uploads
    // pending, after their rt_mesh_upload_finish (a stream sync)
    if (e == cudaSuccess && !pending) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaStreamSynchronize(st);
        rt_set_error("rt_scene_compile: %s", cudaGetErrorString(e));
        return fail(RT_ECUDA);
    }
    // one instance mask for every primitive (the usual case): the build writes it instead of
    // gathering it per leaf
    const uint32_t m0 = n_inst ? inst[0].mask : custom[0].mask;
    s->mask_uniform = 1;
    s->mask_value = m0;
    for (int32_t i = 0; i < n_inst; ++i) s->mask_uniform &= inst[i].mask == m0 && meshes[inst[i].mesh]->nf > 0;
    for (int32_t k = 0; k < n_custom; ++k) s->mask_uniform &= custom[k].mask == m0;
    *out = s;
    return RT_OK;
}

int rt_mesh_info(rt_mesh* m, int64_t* n_vertices, int64_t* n_faces, double* bounds6) {
    RT_CHECK_ARG(m, "mesh is NULL");
    if (m->bounds_dirty && bounds6) {
        unsigned long long r[8];
        RT_CUDA_TRY(cudaSetDevice(m->device));
        RT_CUDA_TRY(cudaMemcpyAsync(r, m->d_red, sizeof r, cudaMemcpyDeviceToHost, m->stream));
        RT_CUDA_TRY(cudaStreamSynchronize(m->stream));
        for (int k = 0; k < 6; ++k) m->bounds[k] = ord2d(r[k]);
        m->bounds_dirty = 0;
    }
    if (n_vertices) *n_vertices = m->nv;
    if (n_faces) *n_faces = m->nf;
    if (bounds6) memcpy(bounds6, m->bounds, sizeof m->bounds);
    return RT_OK;
}

int rt_scene_get_ids(rt_ctx* c, rt_scene* s, int32_t* tri_inst, int32_t* tri_prim, uint32_t* tri_mask,
                     int32_t* tri_material) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const size_t n = (size_t)s->n;
    if (tri_inst) RT_CUDA_TRY(cudaMemcpy(tri_inst, s->tri_inst, 4 * n, cudaMemcpyDeviceToHost));
    if (tri_prim) RT_CUDA_TRY(cudaMemcpy(tri_prim, s->tri_prim, 4 * n, cudaMemcpyDeviceToHost));
    if (tri_mask) RT_CUDA_TRY(cudaMemcpy(tri_mask, s->tri_mask, 4 * n, cudaMemcpyDeviceToHost));
    if (tri_material) {
        std::vector<float4> a(n);
        RT_CUDA_TRY(cudaMemcpy(a.data(), s->tri_attr, sizeof(float4) * n, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i) memcpy(tri_material + i, &a[i].w, 4);
    }
    return RT_OK;
}

void rt_mesh_destroy(rt_mesh* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    if (m->pending) cudaStreamSynchronize(m->stream);   // its copies may still read the host arrays
    void* ptrs[] = {m->faces, m->xform, m->offset, m->verts, m->meta, m->d_red};
    for (void* p : ptrs) rt_free(p, m->stream);
    delete m;
}

}  // extern "C"

extern "C" int rt_scene_get_geometry(rt_ctx* c, rt_scene* s, float* tris9, float* normals3, double* normals64,
                                     double* local_rows9) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(c && s, "NULL argument");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const size_t n = (size_t)s->n;
    if (tris9) RT_CUDA_TRY(cudaMemcpy(tris9, s->tris, sizeof(float) * 9 * n, cudaMemcpyDeviceToHost));
    if (normals3) {
        std::vector<float4> a(n);
        RT_CUDA_TRY(cudaMemcpy(a.data(), s->tri_attr, sizeof(float4) * n, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i) {
            normals3[3 * i] = a[i].x; normals3[3 * i + 1] = a[i].y; normals3[3 * i + 2] = a[i].z;
        }
    }
    if (normals64) {
        RT_CHECK_ARG(s->wnormal64, "scene keeps no float64 world normals");
        RT_CUDA_TRY(cudaMemcpy(normals64, s->wnormal64, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    }
    if (local_rows9) {
        RT_CHECK_ARG(s->lrows64, "scene keeps no float64 local rows");
        RT_CUDA_TRY(cudaMemcpy(local_rows9, s->lrows64, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost));
    }
    return RT_OK;
}
