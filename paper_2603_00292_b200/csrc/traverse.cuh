// traverse.cuh -- the 4-wide closest-hit / any-hit BVH walks, shared by the trace
// kernels (K6), the path-tracing kernels (K7/K8) and the two-level kernels.
//
// Semantics kept from the reference (accel.py:575-653, 762-849; geometry.py:219-330):
//   two-sided triangles, inclusive edges, t in [tmin, tmax] inclusive,
//   u = weight of v1, v = weight of v2, ties -> lowest (instance, prim), i.e.
//   the lowest flat triangle id, instance mask AND ray mask != 0.
// Arithmetic is fp32: a watertight ray/triangle test (Woop, Benthin, Wald 2013)
// with a double-precision fallback for exactly-zero edge functions, and a
// conservative slab test (safe reciprocal, tfar widened by a few ulps, Ize 2013)
// so that culling never drops a box whose triangle the test would accept.
#pragma once
#include "rt_common.cuh"

#ifndef RT_FMA_SLABS
#define RT_FMA_SLABS 1
#endif

// One BVH4 node (128 B, 128-B aligned) as four 256-bit read-only loads (sm_100's
// LDG.E.256) instead of eight 128-bit ones.
#ifndef RT_LDG256
#define RT_LDG256 1
#endif
__device__ __forceinline__ void ldg_pair(const float4* p, float4& a, float4& b) {
#if RT_LDG256
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
#else
    a = __ldg(p);
    b = __ldg(p + 1);
#endif
}
#define RT_LOAD_NODE4(q)                       \
    float4 l0, h0, l1, h1, l2, h2, l3, h3;     \
    ldg_pair((q), l0, h0);                     \
    ldg_pair((q) + 2, l1, h1);                 \
    ldg_pair((q) + 4, l2, h2);                 \
    ldg_pair((q) + 6, l3, h3)

struct RayPre {
    float ox, oy, oz, tmin;
    float dx, dy, dz;          // only the sphere test reads these (dead code for triangle walks)
    float ix, iy, iz;          // safe 1/d
#if RT_FMA_SLABS
    float blx, bly, blz;       // slab plane bias of the lo / hi plane per axis: -o/d -+ e
    float bhx, bhy, bhz;
#endif
    // watertight shear: A' = M (v - o); rows of M
    float m00, m01, m02, m10, m11, m12, m20, m21, m22;
};

__device__ __forceinline__ float safe_rcp(float d) {
    const float eps = 1e-20f;
    return 1.0f / (fabsf(d) > eps ? d : copysignf(eps, d));
}

__device__ __forceinline__ void ray_setup(RayPre& R, float ox, float oy, float oz, float dx, float dy, float dz,
                                          float tmin) {
    R.ox = ox; R.oy = oy; R.oz = oz; R.tmin = tmin;
    R.dx = dx; R.dy = dy; R.dz = dz;
    R.ix = safe_rcp(dx); R.iy = safe_rcp(dy); R.iz = safe_rcp(dz);
#if RT_FMA_SLABS
    {
        // plane distance t = c * (1/d) + (-o/d): one FFMA per plane.  Its error is
        // ~ulp(|o/d|) absolute (the rounded -o/d) + ~ulp(|t|) relative (the FFMA);
        // the absolute part is absorbed PER AXIS by moving the near plane down and
        // the far plane up by e = |o/d| * 2^-21 (a per-ray bound would disable all
        // culling for near-axis rays), the relative part by the tfar widening below
        const float ax = __fmul_rn(ox, R.ix), ay = __fmul_rn(oy, R.iy), az = __fmul_rn(oz, R.iz);
        const float ex = fabsf(ax) * 0x1p-21f, ey = fabsf(ay) * 0x1p-21f, ez = fabsf(az) * 0x1p-21f;
        // for 1/d > 0 the lo plane is the near one
        R.blx = R.ix >= 0.f ? -ax - ex : -ax + ex;  R.bhx = R.ix >= 0.f ? -ax + ex : -ax - ex;
        R.bly = R.iy >= 0.f ? -ay - ey : -ay + ey;  R.bhy = R.iy >= 0.f ? -ay + ey : -ay - ey;
        R.blz = R.iz >= 0.f ? -az - ez : -az + ez;  R.bhz = R.iz >= 0.f ? -az + ez : -az - ez;
    }
#endif
    // kz = argmax |d|, kx = (kz+1)%3, ky = (kx+1)%3; swap kx,ky if d[kz] < 0
    float ax = fabsf(dx), ay = fabsf(dy), az = fabsf(dz);
    int kz = (ax > ay) ? (ax > az ? 0 : 2) : (ay > az ? 1 : 2);
    int kx = kz == 2 ? 0 : kz + 1;
    int ky = kx == 2 ? 0 : kx + 1;
    float dkz = kz == 0 ? dx : (kz == 1 ? dy : dz);
    if (dkz < 0.0f) { int t = kx; kx = ky; ky = t; }
    float dkx = kx == 0 ? dx : (kx == 1 ? dy : dz);
    float dky = ky == 0 ? dx : (ky == 1 ? dy : dz);
    float sz = 1.0f / dkz, sx = dkx * sz, sy = dky * sz;
    // row x: e_kx - sx e_kz ; row y: e_ky - sy e_kz ; row z: sz e_kz
    R.m00 = (kx == 0) ? 1.f : (kz == 0 ? -sx : 0.f);
    R.m01 = (kx == 1) ? 1.f : (kz == 1 ? -sx : 0.f);
    R.m02 = (kx == 2) ? 1.f : (kz == 2 ? -sx : 0.f);
    R.m10 = (ky == 0) ? 1.f : (kz == 0 ? -sy : 0.f);
    R.m11 = (ky == 1) ? 1.f : (kz == 1 ? -sy : 0.f);
    R.m12 = (ky == 2) ? 1.f : (kz == 2 ? -sy : 0.f);
    R.m20 = (kz == 0) ? sz : 0.f;
    R.m21 = (kz == 1) ? sz : 0.f;
    R.m22 = (kz == 2) ? sz : 0.f;
}

// packed fp32x2 FMA (sm_100 FFMA2): two independent correctly rounded FMAs in one
// instruction, bit-identical to two FFMAs
#ifndef RT_BOX_FFMA2
#define RT_BOX_FFMA2 0
#endif
__device__ __forceinline__ void ffma2(float ax, float ay, float bx, float by, float cx, float cy, float& dx,
                                      float& dy) {
    asm("{\n\t.reg .b64 pa, pb, pc, pd;\n\t"
        "mov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\tmov.b64 pc, {%6, %7};\n\t"
        "fma.rn.f32x2 pd, pa, pb, pc;\n\tmov.b64 {%0, %1}, pd;\n\t}"
        : "=f"(dx), "=f"(dy)
        : "f"(ax), "f"(ay), "f"(bx), "f"(by), "f"(cx), "f"(cy));
}

// slab test of one child box against [tmin, tmax]; returns entry distance or +inf on miss
__device__ __forceinline__ float box_enter(const RayPre& R, float lox, float hix, float loy, float hiy, float loz,
                                           float hiz, float tmax) {
    // (lo - o) * (1/d): each slab distance carries at most ~2 ulp of RELATIVE
    // error, so widening tfar by a few ulp keeps the test conservative (Ize 2013)
    // and never culls a box the reference would enter.  (The one-FFMA form
    // lo/d - o/d has an ABSOLUTE error ~ulp(|o/d|): bounding it per ray removes
    // all culling for rays with a near-zero direction component -- measured:
    // 54K node fetches for such a ray on the 10M soup -- and bounding it per axis
    // costs as many instructions as this form.)
#if RT_FMA_SLABS && RT_BOX_FFMA2
    // (x, y) planes as packed pairs: a node slot holds (lo.x, lo.y, lo.z, id), (hi.x, hi.y, hi.z, -),
    // so (lo.x, lo.y) and (hi.x, hi.y) are register pairs straight from the 256-bit loads
    float tx0, ty0, tx1, ty1;
    ffma2(lox, loy, R.ix, R.iy, R.blx, R.bly, tx0, ty0);
    ffma2(hix, hiy, R.ix, R.iy, R.bhx, R.bhy, tx1, ty1);
    float tz0 = __fmaf_rn(loz, R.iz, R.blz), tz1 = __fmaf_rn(hiz, R.iz, R.bhz);
#elif RT_FMA_SLABS
    float tx0 = __fmaf_rn(lox, R.ix, R.blx), tx1 = __fmaf_rn(hix, R.ix, R.bhx);
    float ty0 = __fmaf_rn(loy, R.iy, R.bly), ty1 = __fmaf_rn(hiy, R.iy, R.bhy);
    float tz0 = __fmaf_rn(loz, R.iz, R.blz), tz1 = __fmaf_rn(hiz, R.iz, R.bhz);
#else
    float tx0 = __fmul_rn(__fsub_rn(lox, R.ox), R.ix), tx1 = __fmul_rn(__fsub_rn(hix, R.ox), R.ix);
    float ty0 = __fmul_rn(__fsub_rn(loy, R.oy), R.iy), ty1 = __fmul_rn(__fsub_rn(hiy, R.oy), R.iy);
    float tz0 = __fmul_rn(__fsub_rn(loz, R.oz), R.iz), tz1 = __fmul_rn(__fsub_rn(hiz, R.oz), R.iz);
#endif
    float tn = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), R.tmin));
    float tf = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tmax));
    tf = fmaf(tf, 1.0000008f, 1e-30f);
    return (tn <= tf) ? tn : INFINITY;
}

__device__ __forceinline__ void shear(const RayPre& R, float vx, float vy, float vz, float& X, float& Y, float& Z) {
    float ax = vx - R.ox, ay = vy - R.oy, az = vz - R.oz;
    X = fmaf(R.m00, ax, fmaf(R.m01, ay, R.m02 * az));
    Y = fmaf(R.m10, ax, fmaf(R.m11, ay, R.m12 * az));
    Z = fmaf(R.m20, ax, fmaf(R.m21, ay, R.m22 * az));
}

// edge function without FMA contraction (exact antisymmetry between neighbours)
__device__ __forceinline__ float edge_fn(float ax, float ay, float bx, float by) {
    return __fsub_rn(__fmul_rn(ax, by), __fmul_rn(ay, bx));
}
// exact-zero fallback in double (products of fp32 are exact in fp64)
static __device__ __noinline__ void edge_fn_f64(float Ax, float Ay, float Bx, float By, float Cx, float Cy, float& U,
                                         float& V, float& W) {
    U = (float)((double)Cx * (double)By - (double)Cy * (double)Bx);
    V = (float)((double)Ax * (double)Cy - (double)Ay * (double)Cx);
    W = (float)((double)Bx * (double)Ay - (double)By * (double)Ax);
}

// watertight two-sided test; on success updates (t, id, u, v)
__device__ __forceinline__ bool tri_test(const RayPre& R, const float4 a, const float4 b, const float4 c, float& best_t,
                                         int& best_id, float& bu, float& bv) {
    float Ax, Ay, Az, Bx, By, Bz, Cx, Cy, Cz;
    shear(R, a.x, a.y, a.z, Ax, Ay, Az);
    shear(R, b.x, b.y, b.z, Bx, By, Bz);
    shear(R, c.x, c.y, c.z, Cx, Cy, Cz);
    float U = edge_fn(Cx, Cy, Bx, By);    // Cx*By - Cy*Bx  -> weight of v0
    float V = edge_fn(Ax, Ay, Cx, Cy);    // Ax*Cy - Ay*Cx  -> weight of v1
    float W = edge_fn(Bx, By, Ax, Ay);    // Bx*Ay - By*Ax  -> weight of v2
    if (U == 0.0f || V == 0.0f || W == 0.0f) [[unlikely]]
        edge_fn_f64(Ax, Ay, Bx, By, Cx, Cy, U, V, W);
    if ((U < 0.f || V < 0.f || W < 0.f) && (U > 0.f || V > 0.f || W > 0.f)) return false;
    float det = U + V + W;
    if (det == 0.0f) return false;
    float T = fmaf(U, Az, fmaf(V, Bz, W * Cz));
    float rdet = 1.0f / det;
    float t = T * rdet;
    if (!(t >= R.tmin) || !(t <= best_t)) return false;
    int id = __float_as_int(a.w);
    if (t == best_t && id >= best_id) return false;
    best_t = t;
    best_id = id;
    bu = V * rdet;
    bv = W * rdet;
    return true;
}

// ---- custom primitives: spheres (accel.py:366-423 sphere_intersector; geometry.py:334-363) ----
// A sphere is its own instance (scene.py:101-112) whose single primitive sits in the
// flat primitive list after every triangle: flat ids >= base are spheres, and the
// leaf record holds the instance's world AABB.  rows: 16 doubles per sphere =
// the instance inverse 3x4 (row-major), local center xyz, radius.  The test runs
// in float64 exactly as the reference: ray to local space (accel.py:804-809, the
// direction keeps its length so t is the world t), stable quadratic solve.
// mode 1 = no intersector registered for (sphere, ray type): reaching a sphere
// leaf raises the reference's RegistryError (accel.py:800-803) via *err.
struct SphereView {
    const double* rows;
    int base;          // first sphere flat id (== n: no spheres)
    int mode;          // 0 intersect, 1 error on reach
    int* err;
};

__device__ __forceinline__ void sphere_local(const double* m, double ox, double oy, double oz, double dx, double dy,
                                             double dz, double lo[3], double ld[3]) {
    lo[0] = m[0] * ox + m[1] * oy + m[2] * oz + m[3];
    lo[1] = m[4] * ox + m[5] * oy + m[6] * oz + m[7];
    lo[2] = m[8] * ox + m[9] * oy + m[10] * oz + m[11];
    ld[0] = m[0] * dx + m[1] * dy + m[2] * dz;
    ld[1] = m[4] * dx + m[5] * dy + m[6] * dz;
    ld[2] = m[8] * dx + m[9] * dy + m[10] * dz;
}

// geometry.py:334-363 _sphere_hit in float64 on a local ray (no FMA contraction:
// explicit _rn ops); returns t or -1
__device__ __forceinline__ double sphere_solve_f64(const double o[3], const double d[3], double cx, double cy,
                                                   double cz, double r, double t_min, double t_max) {
    const double lx = __dsub_rn(o[0], cx), ly = __dsub_rn(o[1], cy), lz = __dsub_rn(o[2], cz);
    const double a = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2]));
    const double b = __dmul_rn(2.0, __dadd_rn(__dadd_rn(__dmul_rn(lx, d[0]), __dmul_rn(ly, d[1])), __dmul_rn(lz, d[2])));
    const double c = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(lx, lx), __dmul_rn(ly, ly)), __dmul_rn(lz, lz)),
                               __dmul_rn(r, r));
    const double disc = __dsub_rn(__dmul_rn(b, b), __dmul_rn(__dmul_rn(4.0, a), c));
    if (disc < 0.0) return -1.0;
    const double sq = sqrt(disc);
    const double q = __dmul_rn(-0.5, __dadd_rn(b, copysign(sq, b)));
    double t0, t1;
    if (q == 0.0) { t0 = 0.0; t1 = 0.0; }
    else { t0 = __ddiv_rn(q, a); t1 = __ddiv_rn(c, q); }
    if (t0 > t1) { const double tt = t0; t0 = t1; t1 = tt; }
    double t = t0;
    if (t < t_min || t > t_max) {
        t = t1;
        if (t < t_min || t > t_max) return -1.0;
    }
    return t;
}

// accel.py:804-809 world -> local in float64, the reference's operation order
__device__ __forceinline__ void to_local_f64(const double* m, double ox, double oy, double oz, double dx, double dy,
                                             double dz, double o[3], double d[3]) {
    o[0] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[0], ox), __dmul_rn(m[1], oy)), __dmul_rn(m[2], oz)), m[3]);
    o[1] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[4], ox), __dmul_rn(m[5], oy)), __dmul_rn(m[6], oz)), m[7]);
    o[2] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[8], ox), __dmul_rn(m[9], oy)), __dmul_rn(m[10], oz)), m[11]);
    d[0] = __dadd_rn(__dadd_rn(__dmul_rn(m[0], dx), __dmul_rn(m[1], dy)), __dmul_rn(m[2], dz));
    d[1] = __dadd_rn(__dadd_rn(__dmul_rn(m[4], dx), __dmul_rn(m[5], dy)), __dmul_rn(m[6], dz));
    d[2] = __dadd_rn(__dadd_rn(__dmul_rn(m[8], dx), __dmul_rn(m[9], dy)), __dmul_rn(m[10], dz));
}

// geometry.py:219-275 _tri_hit in float64, the reference's expressions in its order (each
// operation correctly rounded: no contraction); t < 0 = rejected.  V: the vertex type (fp32
// world rows of a flat scene, or a BLAS's float64 local rows)
template <typename V>
__device__ __forceinline__ double tri_hit_f64(const double o[3], const double d[3], double tmin, double tmax,
                                              const V* __restrict__ v9, double& ou, double& ov) {
    const double ax = v9[0], ay = v9[1], az = v9[2], bx = v9[3], by = v9[4], bz = v9[5];
    const double cx = v9[6], cy = v9[7], cz = v9[8];
    const double e0x = __dsub_rn(bx, ax), e0y = __dsub_rn(by, ay), e0z = __dsub_rn(bz, az);
    const double e1x = __dsub_rn(cx, bx), e1y = __dsub_rn(cy, by), e1z = __dsub_rn(cz, bz);
    const double nx = __dsub_rn(__dmul_rn(e0y, e1z), __dmul_rn(e0z, e1y));
    const double ny = __dsub_rn(__dmul_rn(e0z, e1x), __dmul_rn(e0x, e1z));
    const double nz = __dsub_rn(__dmul_rn(e0x, e1y), __dmul_rn(e0y, e1x));
    const double denom = __dadd_rn(__dadd_rn(__dmul_rn(nx, d[0]), __dmul_rn(ny, d[1])), __dmul_rn(nz, d[2]));
    if (denom == 0.0) return -1.0;
    const double num = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(ax, o[0]), nx), __dmul_rn(__dsub_rn(ay, o[1]), ny)),
                                 __dmul_rn(__dsub_rn(az, o[2]), nz));
    const double t = __ddiv_rn(num, denom);
    if (!isfinite(t) || t < tmin || t > tmax) return -1.0;
    const double px = __dadd_rn(o[0], __dmul_rn(d[0], t)), py = __dadd_rn(o[1], __dmul_rn(d[1], t)),
                 pz = __dadd_rn(o[2], __dmul_rn(d[2], t));
    auto edge = [&](double qx, double qy, double qz, double fx, double fy, double fz) {
        const double wx = __dsub_rn(px, qx), wy = __dsub_rn(py, qy), wz = __dsub_rn(pz, qz);
        return __dadd_rn(__dadd_rn(__dmul_rn(nx, __dsub_rn(__dmul_rn(fy, wz), __dmul_rn(fz, wy))),
                                   __dmul_rn(ny, __dsub_rn(__dmul_rn(fz, wx), __dmul_rn(fx, wz)))),
                         __dmul_rn(nz, __dsub_rn(__dmul_rn(fx, wy), __dmul_rn(fy, wx))));
    };
    const double ea = edge(ax, ay, az, e0x, e0y, e0z);
    const double eb = edge(bx, by, bz, e1x, e1y, e1z);
    const double ec = edge(cx, cy, cz, __dsub_rn(ax, cx), __dsub_rn(ay, cy), __dsub_rn(az, cz));
    if (ea < 0.0 || eb < 0.0 || ec < 0.0) return -1.0;
    const double sum = __dadd_rn(__dadd_rn(ea, eb), ec);
    if (sum == 0.0) return -1.0;
    ou = __ddiv_rn(ec, sum);
    ov = __ddiv_rn(ea, sum);
    return t;
}

// geometry.py:334-363 _sphere_hit in float64 on the world ray of a sphere instance
static __device__ __noinline__ double sphere_hit_f64(const double* __restrict__ row, float fox, float foy, float foz,
                                                     float fdx, float fdy, float fdz, double t_min, double t_max) {
    double m[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) m[k] = __ldg(row + k);
    double o[3], d[3];
    to_local_f64(m, fox, foy, foz, fdx, fdy, fdz, o, d);
    return sphere_solve_f64(o, d, __ldg(row + 12), __ldg(row + 13), __ldg(row + 14), __ldg(row + 15), t_min, t_max);
}

// world normal of a sphere hit: local (p - c) / r through the inverse transpose,
// renormalised (geometry.py:360-363, accel.py:843-847), float64
static __device__ __noinline__ float3 sphere_normal(const double* __restrict__ row, float fox, float foy, float foz,
                                                    float fdx, float fdy, float fdz, float t) {
    double m[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) m[k] = __ldg(row + k);
    double o[3], d[3];
    sphere_local(m, fox, foy, foz, fdx, fdy, fdz, o, d);
    const double cx = __ldg(row + 12), cy = __ldg(row + 13), cz = __ldg(row + 14), r = __ldg(row + 15);
    const double px = o[0] + d[0] * (double)t, py = o[1] + d[1] * (double)t, pz = o[2] + d[2] * (double)t;
    const double lnx = (px - cx) / r, lny = (py - cy) / r, lnz = (pz - cz) / r;
    const double wx = m[0] * lnx + m[4] * lny + m[8] * lnz;
    const double wy = m[1] * lnx + m[5] * lny + m[9] * lnz;
    const double wz = m[2] * lnx + m[6] * lny + m[10] * lnz;
    const double il = 1.0 / sqrt(wx * wx + wy * wy + wz * wz);
    return make_float3((float)(wx * il), (float)(wy * il), (float)(wz * il));
}

inline SphereView rt_sphere_view(rt_ctx* ctx, rt_scene* s, int mode) {
    SphereView v;
    v.rows = s->spheres;
    v.base = (int)(s->n - s->n_spheres);
    v.mode = mode;
    v.err = ctx->d_error;
    return v;
}

// closest-hit update for a sphere leaf (u = v = 0 for custom primitives, accel.py:621-623)
static __device__ __noinline__ void sphere_closest(const RayPre& R, const SphereView& sv, int id, float& best_t,
                                                   int& best_id, float& bu, float& bv) {
    if (sv.mode) { atomicExch(sv.err, RT_EUNSUPPORTED); return; }
    const double t = sphere_hit_f64(sv.rows + 16 * (int64_t)(id - sv.base), R.ox, R.oy, R.oz, R.dx, R.dy, R.dz,
                                    (double)R.tmin, (double)best_t);
    if (t < 0.0) return;
    const float tf = (float)t;
    if (tf > best_t || (tf == best_t && id >= best_id)) return;
    best_t = tf; best_id = id; bu = 0.0f; bv = 0.0f;
}

static __device__ __noinline__ bool sphere_any(const RayPre& R, const SphereView& sv, int id, float tmax) {
    if (sv.mode) { atomicExch(sv.err, RT_EUNSUPPORTED); return false; }
    return sphere_hit_f64(sv.rows + 16 * (int64_t)(id - sv.base), R.ox, R.oy, R.oz, R.dx, R.dy, R.dz,
                          (double)R.tmin, (double)tmax) >= 0.0;
}

// shading normal of hit `id` (per-triangle reference normal, or the sphere's at t)
template <bool SPH>
__device__ __forceinline__ void hit_normal(const SphereView& sv, int id, const float4 attr, float ox, float oy, float oz,
                                           float dx, float dy, float dz, float t, float& nx, float& ny, float& nz) {
    nx = attr.x; ny = attr.y; nz = attr.z;
    if (SPH && id >= sv.base) {
        const float3 w = sphere_normal(sv.rows + 16 * (int64_t)(id - sv.base), ox, oy, oz, dx, dy, dz, t);
        nx = w.x; ny = w.y; nz = w.z;
    }
}

struct HitRec {
    float t;
    int id;
    float u, v;
};

__device__ __forceinline__ void cswap(float& ta, int& ca, float& tb, int& cb) {
    if (tb < ta) {
        float t = ta; ta = tb; tb = t;
        int c = ca; ca = cb; cb = c;
    }
}

// Traversal stacks.  LocalStack: the whole stack in local memory (L1-resident).
// SmemStack: the first N entries in shared memory (entry k of thread t at
// base[k * STRIDE + t]: a warp touching one depth hits consecutive words), deeper
// entries spill to local memory.
struct LocalStack {
    int2* p;
    __device__ __forceinline__ void put(int i, int2 v) const { p[i] = v; }
    __device__ __forceinline__ int2 get(int i) const { return p[i]; }
};
template <int N, int STRIDE>
struct SmemStack {
    int2* sm;          // shared: this thread's column
    int2* lm;          // local overflow
    __device__ __forceinline__ void put(int i, int2 v) const {
        if (i < N) sm[i * STRIDE] = v;
        else lm[i - N] = v;
    }
    __device__ __forceinline__ int2 get(int i) const { return i < N ? sm[i * STRIDE] : lm[i - N]; }
};

// 4-wide traversal over the BVH4 view (emit.cuh bvh4_collapse_kernel): one
// 112-B node fetch tests 4 child boxes, children visited nearest first, so a
// ray makes about half the dependent node fetches of the binary walk.  Same
// triangle test, tie rule and conservative slab test as trace_ray.  The stack
// holds at most 3 * ceil(height / 2) entries (checked by the caller).
// Walk budget hook: Y::tick() runs before every walk step (node fetch or leaf test); when it
// returns true the walk
// stops and returns h.id == RT_YIELDED (the tile probe of render.cu).  NoYield folds away,
// so trace_ray4 compiles to the plain walk.
#define RT_YIELDED (-2)
struct NoYield {
    __device__ __forceinline__ bool tick() { return false; }
};

template <bool STATS, bool SPH, typename Stack, typename Y>
__device__ __forceinline__ HitRec trace_ray4_y(const float4* __restrict__ bvh4, int root,
                                               const float4* __restrict__ tris, const RayPre& R, float tmax,
                                               uint32_t ray_mask, const Stack& stack, uint32_t& n_tests,
                                               uint32_t& n_visits, const SphereView& sv, Y& y);

template <bool STATS, bool SPH, typename Stack>
__device__ __forceinline__ HitRec trace_ray4(const float4* __restrict__ bvh4, int root,
                                             const float4* __restrict__ tris, const RayPre& R, float tmax,
                                             uint32_t ray_mask, const Stack& stack, uint32_t& n_tests,
                                             uint32_t& n_visits, const SphereView& sv) {
    NoYield y;
    return trace_ray4_y<STATS, SPH>(bvh4, root, tris, R, tmax, ray_mask, stack, n_tests, n_visits, sv, y);
}

template <bool STATS, bool SPH, typename Stack, typename Y>
__device__ __forceinline__ HitRec trace_ray4_y(const float4* __restrict__ bvh4, int root,
                                               const float4* __restrict__ tris, const RayPre& R, float tmax,
                                               uint32_t ray_mask, const Stack& stack, uint32_t& n_tests,
                                               uint32_t& n_visits, const SphereView& sv, Y& y) {
    HitRec h;
    h.t = tmax; h.id = -1; h.u = 0.f; h.v = 0.f;
    // stack entries carry the child's entry distance: a popped entry that lies
    // beyond the closest hit found since it was pushed is skipped (leaf children
    // would otherwise be tested without re-culling)
    int sp = 0;
    stack.put(0, make_int2(RT_SENTINEL, 0));
    int node = root;
    while (node != RT_SENTINEL) {
        if (y.tick()) {
            h.id = RT_YIELDED;
            return h;
        }
        if (node >= 0) {
            // 4 slots of (lo.xyz, id), (hi.xyz, -)
            const float4* q = bvh4 + 8 * node;
            RT_LOAD_NODE4(q);
            if (STATS) ++n_visits;
            float t0 = box_enter(R, l0.x, h0.x, l0.y, h0.y, l0.z, h0.z, h.t);
            float t1 = box_enter(R, l1.x, h1.x, l1.y, h1.y, l1.z, h1.z, h.t);
            float t2 = box_enter(R, l2.x, h2.x, l2.y, h2.y, l2.z, h2.z, h.t);
            float t3 = box_enter(R, l3.x, h3.x, l3.y, h3.y, l3.z, h3.z, h.t);
            int c0 = __float_as_int(l0.w), c1 = __float_as_int(l1.w), c2 = __float_as_int(l2.w),
                c3 = __float_as_int(l3.w);
            cswap(t0, c0, t1, c1);
            cswap(t2, c2, t3, c3);
            cswap(t0, c0, t2, c2);
            cswap(t1, c1, t3, c3);
            cswap(t1, c1, t2, c2);
            if (t3 != INFINITY) stack.put(++sp, make_int2(c3, __float_as_int(t3)));
            if (t2 != INFINITY) stack.put(++sp, make_int2(c2, __float_as_int(t2)));
            if (t1 != INFINITY) stack.put(++sp, make_int2(c1, __float_as_int(t1)));
            if (t0 != INFINITY) {
                node = c0;
                continue;
            }
        } else {
            const float4* tp = tris + 3 * (~node);
            const float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
            if (STATS) ++n_tests;
            if (__float_as_uint(b.w) & ray_mask) {
                if (!SPH || __float_as_int(a.w) < sv.base) tri_test(R, a, b, c, h.t, h.id, h.u, h.v);
                else sphere_closest(R, sv, __float_as_int(a.w), h.t, h.id, h.u, h.v);
            }
        }
        // pop, dropping entries entered beyond the current closest hit (the box
        // test is inclusive and widened, so ties at t are kept)
        while (true) {
            const int2 e = stack.get(sp--);
            node = e.x;
            if (node == RT_SENTINEL || __int_as_float(e.y) <= fmaf(h.t, 1.0000008f, 1e-30f)) break;
        }
    }
    if (h.id < 0) h.t = -1.0f;
    return h;
}

// watertight test for any-hit: t in [tmin, tmax] inclusive, no closest-t logic
__device__ __forceinline__ bool tri_any(const RayPre& R, const float4 a, const float4 b, const float4 c, float tmax) {
    float best = tmax;
    int id = -1;
    float u, v;
    // tri_test accepts t <= best with (t < best or lower id); with id = -1 a hit
    // exactly at tmax is rejected, so test against a slightly larger bound and
    // re-check inclusively
    best = nextafterf(tmax, INFINITY);
    if (!tri_test(R, a, b, c, best, id, u, v)) return false;
    return best <= tmax;
}

// Any-hit (accel.py:656-699, 852-895): the first accepted intersection in
// [tmin, tmax] ends the walk; children are visited in slot order (no sort).
template <bool SPH>
__device__ __forceinline__ bool trace_any4(const float4* __restrict__ bvh4, int root, const float4* __restrict__ tris,
                                           const RayPre& R, float tmax, uint32_t ray_mask, int* stack,
                                           const SphereView& sv) {
    int sp = 0;
    stack[0] = RT_SENTINEL;
    int node = root;
    while (node != RT_SENTINEL) {
        if (node >= 0) {
            const float4* q = bvh4 + 8 * node;
            RT_LOAD_NODE4(q);
            const bool b0 = box_enter(R, l0.x, h0.x, l0.y, h0.y, l0.z, h0.z, tmax) != INFINITY;
            const bool b1 = box_enter(R, l1.x, h1.x, l1.y, h1.y, l1.z, h1.z, tmax) != INFINITY;
            const bool b2 = box_enter(R, l2.x, h2.x, l2.y, h2.y, l2.z, h2.z, tmax) != INFINITY;
            const bool b3 = box_enter(R, l3.x, h3.x, l3.y, h3.y, l3.z, h3.z, tmax) != INFINITY;
            if (b3) stack[++sp] = __float_as_int(l3.w);
            if (b2) stack[++sp] = __float_as_int(l2.w);
            if (b1) stack[++sp] = __float_as_int(l1.w);
            if (b0) stack[++sp] = __float_as_int(l0.w);
        } else {
            const float4* tp = tris + 3 * (~node);
            const float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
            if (__float_as_uint(b.w) & ray_mask) {
                if ((!SPH || __float_as_int(a.w) < sv.base) ? tri_any(R, a, b, c, tmax)
                                                            : sphere_any(R, sv, __float_as_int(a.w), tmax))
                    return true;
            }
        }
        node = stack[sp--];
    }
    return false;
}

// Stack of the 4-wide walk: at most 3 pushes per BVH4 level and ceil(h/2) levels
// for a binary tree of height h <= RT_STACK - 1 (the depth limit the build enforces).
#define RT_STACK4 (3 * (RT_STACK / 2) + 4)


// ---- generic 4-wide walks with a leaf callback (two-level traversal, tlas.cu) ----
// Same node layout, slab test, nearest-first order and pop culling as
// trace_ray4; leaf(k) handles leaf k and may lower best_t.
template <bool STATS, typename Leaf>
__device__ __forceinline__ void walk4(const float4* __restrict__ bvh4, int root, const RayPre& R, float& best_t,
                                      int2* stack, uint32_t& n_visits, Leaf&& leaf) {
    int sp = 0;
    stack[0] = make_int2(RT_SENTINEL, 0);
    int node = root;
    while (node != RT_SENTINEL) {
        if (node >= 0) {
            const float4* q = bvh4 + 8 * node;
            RT_LOAD_NODE4(q);
            if (STATS) ++n_visits;
            float t0 = box_enter(R, l0.x, h0.x, l0.y, h0.y, l0.z, h0.z, best_t);
            float t1 = box_enter(R, l1.x, h1.x, l1.y, h1.y, l1.z, h1.z, best_t);
            float t2 = box_enter(R, l2.x, h2.x, l2.y, h2.y, l2.z, h2.z, best_t);
            float t3 = box_enter(R, l3.x, h3.x, l3.y, h3.y, l3.z, h3.z, best_t);
            int c0 = __float_as_int(l0.w), c1 = __float_as_int(l1.w), c2 = __float_as_int(l2.w),
                c3 = __float_as_int(l3.w);
            cswap(t0, c0, t1, c1);
            cswap(t2, c2, t3, c3);
            cswap(t0, c0, t2, c2);
            cswap(t1, c1, t3, c3);
            cswap(t1, c1, t2, c2);
            if (t3 != INFINITY) stack[++sp] = make_int2(c3, __float_as_int(t3));
            if (t2 != INFINITY) stack[++sp] = make_int2(c2, __float_as_int(t2));
            if (t1 != INFINITY) stack[++sp] = make_int2(c1, __float_as_int(t1));
            if (t0 != INFINITY) {
                node = c0;
                continue;
            }
        } else {
            leaf(~node);
        }
        while (true) {
            const int2 e = stack[sp--];
            node = e.x;
            if (node == RT_SENTINEL || __int_as_float(e.y) <= fmaf(best_t, 1.0000008f, 1e-30f)) break;
        }
    }
}

// any-hit walk: leaf(k) returns true to stop
template <typename Leaf>
__device__ __forceinline__ bool walk_any4(const float4* __restrict__ bvh4, int root, const RayPre& R, float tmax,
                                          int* stack, Leaf&& leaf) {
    int sp = 0;
    stack[0] = RT_SENTINEL;
    int node = root;
    while (node != RT_SENTINEL) {
        if (node >= 0) {
            const float4* q = bvh4 + 8 * node;
            RT_LOAD_NODE4(q);
            if (box_enter(R, l3.x, h3.x, l3.y, h3.y, l3.z, h3.z, tmax) != INFINITY) stack[++sp] = __float_as_int(l3.w);
            if (box_enter(R, l2.x, h2.x, l2.y, h2.y, l2.z, h2.z, tmax) != INFINITY) stack[++sp] = __float_as_int(l2.w);
            if (box_enter(R, l1.x, h1.x, l1.y, h1.y, l1.z, h1.z, tmax) != INFINITY) stack[++sp] = __float_as_int(l1.w);
            if (box_enter(R, l0.x, h0.x, l0.y, h0.y, l0.z, h0.z, tmax) != INFINITY) stack[++sp] = __float_as_int(l0.w);
        } else if (leaf(~node)) {
            return true;
        }
        node = stack[sp--];
    }
    return false;
}
