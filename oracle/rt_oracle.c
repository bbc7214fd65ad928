/*
 * rt_oracle.c -- CPU ORACLE for the B200 ray-tracing hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2603_00292_b200/)
 * links, loads or calls this file.  It is used by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * `--impl reference` leg as the timed CPU baseline ("kind": "port").
 *
 * Part A restates the reference's float64 algorithm for the hot path
 * (pkg/src/pathtrace, a numba CPU library) operation for operation, so that
 * the result is bit-identical to the reference on the same inputs:
 *   - _tri_hit            geometry.py:219-275
 *   - _sphere_hit / sphere_intersector   geometry.py:334-363, accel.py:396-401
 *   - _aabb_hit           geometry.py:278-330
 *   - _build_bvh (binned SAH / median)   accel.py:68-187
 *   - _blas_closest / _tlas_closest      accel.py:575-653, 762-849
 *   - _blas_any / _tlas_any              accel.py:656-699, 852-895
 *   - _mix64/_pcg_next/_pcg_init/_stream_for/_uniform   sampling.py:38-79
 *   - _cosine_dir / _onb                 sampling.py:144-151, 175-186
 *   - _primary_dir                       camera.py:81-97
 *   - _geom_term                         integrators.py:99-115
 *   - _sample_eye/_sample_ao/_sample_pt/_sample_ptnee  integrators.py:129-331
 *   - _render_chunk / render_frame worker split        integrators.py:334-379, 426-473
 * Compiled with -ffp-contract=off (numba/LLVM without fastmath does not
 * contract), so every double operation rounds exactly as in the reference.
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 *
 * Part B is the CPU restatement of the LBVH the GPU builds.  The reference has
 * no LBVH; the frozen choices of SURVEY.md section 8(c) are
 * implemented here (Karras 2012): fp32 centroid bounds, 30/63-bit Morton
 * codes without FMA, stable (key, index) sort, Karras split with the index
 * fallback for equal keys, fp32 min/max refit.  The GPU LBVH must match it
 * bit for bit (tests/test_gpu_lbvh.py).  Its topology parity is pinned by this
 * restatement only; the resulting BVH is validated through the reference's
 * traversal (tests/test_oracle_golden.py::test_lbvh_through_reference_traversal).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ======================================================================== */
/* Part A.1  scalar kernels (geometry.py)                                   */
/* ======================================================================== */

/* geometry.py:219-275  _tri_hit; returns t (<0 = miss) and u, v, n */
static inline double tri_hit(double ox, double oy, double oz, double dx, double dy, double dz,
                             double t_min, double t_max,
                             double ax, double ay, double az, double bx, double by, double bz,
                             double cx, double cy, double cz,
                             double* ou, double* ov, double* onx, double* ony, double* onz)
{
    double e0x = bx - ax, e0y = by - ay, e0z = bz - az;
    double e1x = cx - bx, e1y = cy - by, e1z = cz - bz;
    double nx = e0y * e1z - e0z * e1y;
    double ny = e0z * e1x - e0x * e1z;
    double nz = e0x * e1y - e0y * e1x;
    double denom = nx * dx + ny * dy + nz * dz;
    if (denom == 0.0) return -1.0;
    double t = ((ax - ox) * nx + (ay - oy) * ny + (az - oz) * nz) / denom;
    if (!isfinite(t)) return -1.0;
    if (t < t_min || t > t_max) return -1.0;
    double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
    double wx = px - ax, wy = py - ay, wz = pz - az;
    double ea = nx * (e0y * wz - e0z * wy) + ny * (e0z * wx - e0x * wz) + nz * (e0x * wy - e0y * wx);
    wx = px - bx; wy = py - by; wz = pz - bz;
    double eb = nx * (e1y * wz - e1z * wy) + ny * (e1z * wx - e1x * wz) + nz * (e1x * wy - e1y * wx);
    double e2x = ax - cx, e2y = ay - cy, e2z = az - cz;
    wx = px - cx; wy = py - cy; wz = pz - cz;
    double ec = nx * (e2y * wz - e2z * wy) + ny * (e2z * wx - e2x * wz) + nz * (e2x * wy - e2y * wx);
    if (ea < 0.0 || eb < 0.0 || ec < 0.0) return -1.0;
    double s = ea + eb + ec;
    if (s == 0.0) return -1.0;
    *ou = ec / s;
    *ov = ea / s;
    double nlen = sqrt(nx * nx + ny * ny + nz * nz);
    *onx = nx / nlen; *ony = ny / nlen; *onz = nz / nlen;
    return t;
}

/* geometry.py:334-363  _sphere_hit: stable quadratic solve; t < 0 on miss */
static inline double sphere_hit(double ox, double oy, double oz, double dx, double dy, double dz,
                                double t_min, double t_max, double cx, double cy, double cz, double r,
                                double* onx, double* ony, double* onz)
{
    double lx = ox - cx, ly = oy - cy, lz = oz - cz;
    double a = dx * dx + dy * dy + dz * dz;
    double b = 2.0 * (lx * dx + ly * dy + lz * dz);
    double c = lx * lx + ly * ly + lz * lz - r * r;
    double disc = b * b - 4.0 * a * c;
    if (disc < 0.0) return -1.0;
    double sq = sqrt(disc);
    double q = -0.5 * (b + copysign(sq, b));
    double t0, t1;
    if (q == 0.0) { t0 = 0.0; t1 = 0.0; }
    else { t0 = q / a; t1 = c / q; }
    if (t0 > t1) { double tmp = t0; t0 = t1; t1 = tmp; }
    double t = t0;
    if (t < t_min || t > t_max) {
        t = t1;
        if (t < t_min || t > t_max) return -1.0;
    }
    double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
    *onx = (px - cx) / r; *ony = (py - cy) / r; *onz = (pz - cz) / r;
    return t;
}

/* geometry.py:278-330  _aabb_hit, inclusive, containment for infinite 1/d */
static inline int aabb_axis(double o, double inv, double lo, double hi, double* tlo, double* thi)
{
    if (isinf(inv)) {
        if (o < lo || o > hi) return 0;
        return 1;
    }
    double t0 = (lo - o) * inv, t1 = (hi - o) * inv;
    if (t0 > t1) { double tmp = t0; t0 = t1; t1 = tmp; }
    if (t0 > *tlo) *tlo = t0;
    if (t1 < *thi) *thi = t1;
    if (*tlo > *thi) return 0;
    return 1;
}

static inline int aabb_hit(double ox, double oy, double oz, double ix, double iy, double iz,
                           double t_min, double t_max, const double* b)
{
    double tlo = t_min, thi = t_max;
    if (!aabb_axis(ox, ix, b[0], b[3], &tlo, &thi)) return 0;
    if (!aabb_axis(oy, iy, b[1], b[4], &tlo, &thi)) return 0;
    if (!aabb_axis(oz, iz, b[2], b[5], &tlo, &thi)) return 0;
    return 1;
}

ORC_API double orc_tri_hit(const double* ray8, const double* v9, double* out5)
{
    double u = 0, v = 0, nx = 0, ny = 0, nz = 0;
    double t = tri_hit(ray8[0], ray8[1], ray8[2], ray8[3], ray8[4], ray8[5], ray8[6], ray8[7],
                       v9[0], v9[1], v9[2], v9[3], v9[4], v9[5], v9[6], v9[7], v9[8],
                       &u, &v, &nx, &ny, &nz);
    if (t < 0.0) { u = v = nx = ny = nz = 0.0; }
    out5[0] = u; out5[1] = v; out5[2] = nx; out5[3] = ny; out5[4] = nz;
    return t;
}

/* ======================================================================== */
/* Part A.2  top-down BVH build (accel.py:68-187)                           */
/* ======================================================================== */

#define SAH_BINS 16
#define MAX_STACK_DEPTH 64
#define FORCE_MEDIAN_DEPTH 32

typedef struct {
    int64_t n;
    const double* lo;      /* (n,3) prim boxes */
    const double* hi;
    double* cen;           /* (n,3) centroids 0.5*(lo+hi)  accel.py:78 */
    int balanced;
    int max_leaf;
    /* outputs */
    double* bounds;        /* (cap,6) */
    int64_t *left, *right, *count, *axis, *order;
    int64_t cap, nodes, cursor, deepest;
    int err;
    /* scratch */
    int64_t* tmp;          /* n */
    int64_t* bin_id;       /* n */
    double* key;           /* n */
} bvh_builder;

static double box_area(const double* lo, const double* hi)
{
    /* accel.py:61-63  d = max(hi - lo, 0); 2*(d0 d1 + d1 d2 + d2 d0) */
    double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
    d0 = (d0 > 0.0 || isnan(d0)) ? d0 : 0.0;
    d1 = (d1 > 0.0 || isnan(d1)) ? d1 : 0.0;
    d2 = (d2 > 0.0 || isnan(d2)) ? d2 : 0.0;
    return 2.0 * (d0 * d1 + d1 * d2 + d2 * d0);
}

static const double* g_sort_key;
static int cmp_stable(const void* a, const void* b)
{
    int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
    double ki = g_sort_key[i], kj = g_sort_key[j];
    if (ki < kj) return -1;
    if (ki > kj) return 1;
    return (i < j) ? -1 : (i > j);
}

static void centroid_extent(bvh_builder* B, const int64_t* idx, int64_t m, double* cmin, double* ext)
{
    double cmax[3];
    for (int a = 0; a < 3; ++a) { cmin[a] = INFINITY; cmax[a] = -INFINITY; }
    for (int64_t k = 0; k < m; ++k) {
        const double* c = B->cen + 3 * idx[k];
        for (int a = 0; a < 3; ++a) {
            if (c[a] < cmin[a]) cmin[a] = c[a];
            if (c[a] > cmax[a]) cmax[a] = c[a];
        }
    }
    for (int a = 0; a < 3; ++a) ext[a] = cmax[a] - cmin[a];
}

static int argmax3(const double* e)
{
    int ax = 0;
    if (e[1] > e[ax]) ax = 1;
    if (e[2] > e[ax]) ax = 2;
    return ax;
}

/* accel.py:88-96 median_split: stable argsort along the longest centroid axis */
static int median_split(bvh_builder* B, int64_t* idx, int64_t m, int64_t* nl)
{
    double cmin[3], ext[3];
    centroid_extent(B, idx, m, cmin, ext);
    int ax = argmax3(ext);
    int64_t half = m / 2;
    *nl = half;
    if (ext[ax] <= 0.0) return 0;
    /* stable argsort of c[:, ax] over positions 0..m-1 */
    for (int64_t k = 0; k < m; ++k) { B->key[k] = B->cen[3 * idx[k] + ax]; B->tmp[k] = k; }
    g_sort_key = B->key;
    qsort(B->tmp, (size_t)m, sizeof(int64_t), cmp_stable);
    /* idx[srt] */
    for (int64_t k = 0; k < m; ++k) B->bin_id[k] = idx[B->tmp[k]];
    memcpy(idx, B->bin_id, (size_t)m * sizeof(int64_t));
    return ax;
}

/* accel.py:98-144 sah_split; returns 1 and partitions idx in place (stable) */
static int sah_split(bvh_builder* B, int64_t* idx, int64_t m, double node_area, int64_t* nl_out, int* ax_out)
{
    double cb_lo[3], ext[3];
    centroid_extent(B, idx, m, cb_lo, ext);
    int ax = argmax3(ext);
    if (ext[ax] <= 0.0) return 0;
    double scale = (double)SAH_BINS / ext[ax];
    int64_t counts[SAH_BINS] = {0};
    double b_lo[SAH_BINS][3], b_hi[SAH_BINS][3];
    for (int k = 0; k < SAH_BINS; ++k)
        for (int a = 0; a < 3; ++a) { b_lo[k][a] = INFINITY; b_hi[k][a] = -INFINITY; }
    for (int64_t k = 0; k < m; ++k) {
        int64_t p = idx[k];
        double x = (B->cen[3 * p + ax] - cb_lo[ax]) * scale;
        int64_t b = (int64_t)x;               /* astype(int64): truncation */
        if (b > SAH_BINS - 1) b = SAH_BINS - 1;
        B->bin_id[k] = b;
        counts[b]++;
        for (int a = 0; a < 3; ++a) {
            double lo = B->lo[3 * p + a], hi = B->hi[3 * p + a];
            if (lo < b_lo[b][a]) b_lo[b][a] = lo;   /* np.minimum.at */
            if (hi > b_hi[b][a]) b_hi[b][a] = hi;
        }
    }
    double best_cost = INFINITY;
    int best_k = -1;
    double l_lo[3] = {INFINITY, INFINITY, INFINITY}, l_hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    double l_area[SAH_BINS - 1];
    int64_t l_count[SAH_BINS - 1];
    int64_t run = 0;
    for (int k = 0; k < SAH_BINS - 1; ++k) {
        for (int a = 0; a < 3; ++a) {
            if (b_lo[k][a] < l_lo[a]) l_lo[a] = b_lo[k][a];
            if (b_hi[k][a] > l_hi[a]) l_hi[a] = b_hi[k][a];
        }
        l_area[k] = box_area(l_lo, l_hi);
        run += counts[k];
        l_count[k] = run;
    }
    double r_lo[3] = {INFINITY, INFINITY, INFINITY}, r_hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = SAH_BINS - 2; k >= 0; --k) {
        for (int a = 0; a < 3; ++a) {
            if (b_lo[k + 1][a] < r_lo[a]) r_lo[a] = b_lo[k + 1][a];
            if (b_hi[k + 1][a] > r_hi[a]) r_hi[a] = b_hi[k + 1][a];
        }
        int64_t nl = l_count[k], nr = m - nl;
        if (nl == 0 || nr == 0) continue;
        double cost = 1.0 + 1.0 * (l_area[k] * (double)nl + box_area(r_lo, r_hi) * (double)nr) / node_area;
        if (cost <= best_cost) { best_cost = cost; best_k = k; }
    }
    if (best_k < 0 || best_cost >= 1.0 * (double)m) return 0;
    /* idx[mask], idx[~mask] keeping order */
    int64_t nl = 0, nr = 0;
    for (int64_t k = 0; k < m; ++k)
        if (B->bin_id[k] <= best_k) B->tmp[nl++] = idx[k];
    for (int64_t k = 0; k < m; ++k)
        if (B->bin_id[k] > best_k) B->tmp[nl + nr++] = idx[k];
    memcpy(idx, B->tmp, (size_t)m * sizeof(int64_t));
    *nl_out = nl;
    *ax_out = ax;
    return 1;
}

/* accel.py:146-176 build(idx, depth): preorder, leaf <= max_leaf */
static int64_t build_rec(bvh_builder* B, int64_t* idx, int64_t m, int64_t depth)
{
    if (B->err) return 0;
    if (depth > MAX_STACK_DEPTH) { B->err = -2; return 0; }
    if (depth > B->deepest) B->deepest = depth;
    int64_t slot = B->nodes++;
    if (slot >= B->cap) { B->err = -3; return 0; }
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = 0; k < m; ++k) {
        int64_t p = idx[k];
        for (int a = 0; a < 3; ++a) {
            if (B->lo[3 * p + a] < lo[a]) lo[a] = B->lo[3 * p + a];
            if (B->hi[3 * p + a] > hi[a]) hi[a] = B->hi[3 * p + a];
        }
    }
    for (int a = 0; a < 3; ++a) { B->bounds[6 * slot + a] = lo[a]; B->bounds[6 * slot + 3 + a] = hi[a]; }
    B->left[slot] = 0; B->right[slot] = -1; B->count[slot] = 0; B->axis[slot] = 0;
    if (m <= B->max_leaf) {
        B->left[slot] = B->cursor;
        B->count[slot] = m;
        for (int64_t k = 0; k < m; ++k) B->order[B->cursor + k] = idx[k];
        B->cursor += m;
        return slot;
    }
    int done = 0, ax = 0;
    int64_t nl = 0;
    if (B->balanced && depth < FORCE_MEDIAN_DEPTH) {
        double area = box_area(lo, hi);
        if (area > 0.0) done = sah_split(B, idx, m, area, &nl, &ax);
    }
    if (!done) ax = median_split(B, idx, m, &nl);
    B->axis[slot] = ax;
    int64_t l = build_rec(B, idx, nl, depth + 1);
    B->left[slot] = l;
    int64_t r = build_rec(B, idx + nl, m - nl, depth + 1);
    B->right[slot] = r;
    return slot;
}

/* returns number of nodes (>0) or a negative error; cap must be >= 2n */
ORC_API int64_t orc_build_bvh(int64_t n, const double* lo, const double* hi, int balanced, int max_leaf,
                              double* bounds, int64_t* left, int64_t* right, int64_t* count,
                              int64_t* axis, int64_t* order, int64_t cap, int64_t* depth_out)
{
    if (n <= 0) return -1;
    bvh_builder B;
    memset(&B, 0, sizeof B);
    B.n = n; B.lo = lo; B.hi = hi; B.balanced = balanced; B.max_leaf = max_leaf;
    B.bounds = bounds; B.left = left; B.right = right; B.count = count; B.axis = axis; B.order = order;
    B.cap = cap; B.deepest = 1;
    B.cen = (double*)malloc((size_t)n * 3 * sizeof(double));
    B.tmp = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    B.bin_id = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    B.key = (double*)malloc((size_t)n * sizeof(double));
    int64_t* idx = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < 3 * n; ++i) B.cen[i] = 0.5 * (lo[i] + hi[i]);
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    build_rec(&B, idx, n, 1);
    free(B.cen); free(B.tmp); free(B.bin_id); free(B.key); free(idx);
    if (B.err) return B.err;
    *depth_out = B.deepest;
    return B.nodes;
}

/* ======================================================================== */
/* Part A.3  two-level traversal (accel.py TlasBundle + kernels)            */
/* ======================================================================== */

typedef struct {
    /* top level  (accel.py:430-436 TlasBundle fields) */
    const double* t_bounds; const int64_t *t_left, *t_right, *t_count, *t_axis, *t_order;
    const int64_t* i_blas; const uint64_t* i_mask; const double* i_inv; /* (I,3,4) */
    const int64_t *b_node_ofs, *b_prim_ofs, *b_kind, *b_tri_ofs;
    const double* n_bounds; const int64_t *n_left, *n_right, *n_count, *n_axis;
    const int64_t* prim_order; const int64_t* tri_vidx; const double* verts;
    int64_t n_inst;
    /* custom primitives (accel.py:41-43 CUSTOM; sphere_intersector data rows cx cy cz r) */
    const int64_t* b_data_ofs; const double* custom_data;
} orc_bundle;

#define KIND_CUSTOM 1

#define PRIM_SENTINEL ((int64_t)1 << 62)

/* accel.py:575-653 */
static int blas_closest(const orc_bundle* bd, int64_t b, double ox, double oy, double oz,
                        double dx, double dy, double dz, double t_min, double best_t,
                        double* ot, int64_t* oprim, double* onx, double* ony, double* onz,
                        double* ou, double* ov, int64_t* tests, int64_t* visits)
{
    int64_t stack[MAX_STACK_DEPTH];
    int64_t node0 = bd->b_node_ofs[b], prim0 = bd->b_prim_ofs[b], tri0 = bd->b_tri_ofs[b];
    double ix = 1.0 / dx, iy = 1.0 / dy, iz = 1.0 / dz;
    int found = 0;
    double cur_t = best_t;
    int64_t cur_prim = PRIM_SENTINEL;
    double hnx = 0, hny = 0, hnz = 0, hu = 0, hv = 0;
    int sp = 1;
    stack[0] = 0;
    while (sp > 0) {
        sp -= 1;
        int64_t row = node0 + stack[sp];
        *visits += 1;
        if (!aabb_hit(ox, oy, oz, ix, iy, iz, t_min, cur_t, bd->n_bounds + 6 * row)) continue;
        int64_t cnt = bd->n_count[row];
        if (cnt > 0) {
            int64_t first = prim0 + bd->n_left[row];
            for (int64_t k = 0; k < cnt; ++k) {
                int64_t prim = bd->prim_order[first + k];
                *tests += 1;
                double u = 0, v = 0, nx = 0, ny = 0, nz = 0, t;
                if (bd->b_kind[b] == KIND_CUSTOM) {
                    /* accel.py:618-623: _custom_hit(table, slot, data0 + prim, ...), u = v = 0 */
                    const double* S = bd->custom_data + 4 * (bd->b_data_ofs[b] + prim);
                    t = sphere_hit(ox, oy, oz, dx, dy, dz, t_min, cur_t, S[0], S[1], S[2], S[3], &nx, &ny, &nz);
                } else {
                    int64_t tri = tri0 + prim;
                    const double* A = bd->verts + 3 * bd->tri_vidx[3 * tri + 0];
                    const double* Bv = bd->verts + 3 * bd->tri_vidx[3 * tri + 1];
                    const double* C = bd->verts + 3 * bd->tri_vidx[3 * tri + 2];
                    t = tri_hit(ox, oy, oz, dx, dy, dz, t_min, cur_t,
                                A[0], A[1], A[2], Bv[0], Bv[1], Bv[2], C[0], C[1], C[2],
                                &u, &v, &nx, &ny, &nz);
                }
                if (t >= 0.0 && (t < cur_t || (t == cur_t && prim < cur_prim))) {
                    found = 1; cur_t = t; cur_prim = prim;
                    hnx = nx; hny = ny; hnz = nz; hu = u; hv = v;
                }
            }
        } else {
            int64_t ax = bd->n_axis[row];
            double d = ax == 0 ? dx : (ax == 1 ? dy : dz);
            if (d >= 0.0) { stack[sp] = bd->n_right[row]; stack[sp + 1] = bd->n_left[row]; }
            else          { stack[sp] = bd->n_left[row];  stack[sp + 1] = bd->n_right[row]; }
            sp += 2;
        }
    }
    *ot = cur_t; *oprim = cur_prim; *onx = hnx; *ony = hny; *onz = hnz; *ou = hu; *ov = hv;
    return found;
}

/* accel.py:656-699 */
static int blas_any(const orc_bundle* bd, int64_t b, double ox, double oy, double oz,
                    double dx, double dy, double dz, double t_min, double t_max)
{
    int64_t stack[MAX_STACK_DEPTH];
    int64_t node0 = bd->b_node_ofs[b], prim0 = bd->b_prim_ofs[b], tri0 = bd->b_tri_ofs[b];
    double ix = 1.0 / dx, iy = 1.0 / dy, iz = 1.0 / dz;
    int sp = 1;
    stack[0] = 0;
    while (sp > 0) {
        sp -= 1;
        int64_t row = node0 + stack[sp];
        if (!aabb_hit(ox, oy, oz, ix, iy, iz, t_min, t_max, bd->n_bounds + 6 * row)) continue;
        int64_t cnt = bd->n_count[row];
        if (cnt > 0) {
            int64_t first = prim0 + bd->n_left[row];
            for (int64_t k = 0; k < cnt; ++k) {
                int64_t prim = bd->prim_order[first + k];
                double u, v, nx, ny, nz, t;
                if (bd->b_kind[b] == KIND_CUSTOM) {
                    const double* S = bd->custom_data + 4 * (bd->b_data_ofs[b] + prim);
                    t = sphere_hit(ox, oy, oz, dx, dy, dz, t_min, t_max, S[0], S[1], S[2], S[3], &nx, &ny, &nz);
                } else {
                    int64_t tri = tri0 + prim;
                    const double* A = bd->verts + 3 * bd->tri_vidx[3 * tri + 0];
                    const double* Bv = bd->verts + 3 * bd->tri_vidx[3 * tri + 1];
                    const double* C = bd->verts + 3 * bd->tri_vidx[3 * tri + 2];
                    t = tri_hit(ox, oy, oz, dx, dy, dz, t_min, t_max,
                                A[0], A[1], A[2], Bv[0], Bv[1], Bv[2], C[0], C[1], C[2],
                                &u, &v, &nx, &ny, &nz);
                }
                if (t >= 0.0) return 1;
            }
        } else {
            stack[sp] = bd->n_left[row];
            stack[sp + 1] = bd->n_right[row];
            sp += 2;
        }
    }
    return 0;
}

static inline void to_local(const double* m, double ox, double oy, double oz, double dx, double dy, double dz,
                            double* lo, double* ld)
{
    /* accel.py:804-809 */
    lo[0] = m[0] * ox + m[1] * oy + m[2] * oz + m[3];
    lo[1] = m[4] * ox + m[5] * oy + m[6] * oz + m[7];
    lo[2] = m[8] * ox + m[9] * oy + m[10] * oz + m[11];
    ld[0] = m[0] * dx + m[1] * dy + m[2] * dz;
    ld[1] = m[4] * dx + m[5] * dy + m[6] * dz;
    ld[2] = m[8] * dx + m[9] * dy + m[10] * dz;
}

typedef struct {
    double t, nx, ny, nz, u, v;
    int64_t inst, prim, tests, visits;
} orc_hit;

/* accel.py:762-849; returns 1 hit, 0 miss */
static int tlas_closest(const orc_bundle* bd, double ox, double oy, double oz, double dx, double dy, double dz,
                        double t_min, double t_max, uint64_t ray_mask, orc_hit* h)
{
    int64_t tstack[MAX_STACK_DEPTH];
    double best_t = t_max;
    int64_t best_inst = -1, best_prim = -1;
    double lnx = 0, lny = 0, lnz = 0, hu = 0, hv = 0;
    int64_t tests = 0, visits = 0;
    double ix = 1.0 / dx, iy = 1.0 / dy, iz = 1.0 / dz;
    int sp = 1;
    tstack[0] = 0;
    while (sp > 0) {
        sp -= 1;
        int64_t node = tstack[sp];
        visits += 1;
        if (!aabb_hit(ox, oy, oz, ix, iy, iz, t_min, best_t, bd->t_bounds + 6 * node)) continue;
        int64_t cnt = bd->t_count[node];
        if (cnt > 0) {
            int64_t first = bd->t_left[node];
            for (int64_t k = 0; k < cnt; ++k) {
                int64_t inst = bd->t_order[first + k];
                if ((bd->i_mask[inst] & ray_mask) == 0) continue;
                int64_t b = bd->i_blas[inst];
                double lo[3], ld[3];
                to_local(bd->i_inv + 12 * inst, ox, oy, oz, dx, dy, dz, lo, ld);
                double t, nx, ny, nz, u, v;
                int64_t prim;
                int found = blas_closest(bd, b, lo[0], lo[1], lo[2], ld[0], ld[1], ld[2], t_min, best_t,
                                         &t, &prim, &nx, &ny, &nz, &u, &v, &tests, &visits);
                if (found == 1 && (t < best_t || (t == best_t && (inst < best_inst ||
                                                                  (inst == best_inst && prim < best_prim))))) {
                    best_t = t; best_inst = inst; best_prim = prim;
                    lnx = nx; lny = ny; lnz = nz; hu = u; hv = v;
                }
            }
        } else {
            int64_t ax = bd->t_axis[node];
            double d = ax == 0 ? dx : (ax == 1 ? dy : dz);
            if (d >= 0.0) { tstack[sp] = bd->t_right[node]; tstack[sp + 1] = bd->t_left[node]; }
            else          { tstack[sp] = bd->t_left[node];  tstack[sp + 1] = bd->t_right[node]; }
            sp += 2;
        }
    }
    h->tests = tests; h->visits = visits;
    if (best_inst < 0) { h->inst = -1; h->prim = -1; h->t = 0.0; return 0; }
    const double* m = bd->i_inv + 12 * best_inst;
    /* accel.py:843-847  world normal via the inverse transpose */
    double wnx = m[0] * lnx + m[4] * lny + m[8] * lnz;
    double wny = m[1] * lnx + m[5] * lny + m[9] * lnz;
    double wnz = m[2] * lnx + m[6] * lny + m[10] * lnz;
    double inv_len = 1.0 / sqrt(wnx * wnx + wny * wny + wnz * wnz);
    h->t = best_t; h->inst = best_inst; h->prim = best_prim;
    h->nx = wnx * inv_len; h->ny = wny * inv_len; h->nz = wnz * inv_len;
    h->u = hu; h->v = hv;
    return 1;
}

/* accel.py:852-895 */
static int tlas_any(const orc_bundle* bd, double ox, double oy, double oz, double dx, double dy, double dz,
                    double t_min, double t_max, uint64_t ray_mask)
{
    int64_t tstack[MAX_STACK_DEPTH];
    double ix = 1.0 / dx, iy = 1.0 / dy, iz = 1.0 / dz;
    int sp = 1;
    tstack[0] = 0;
    while (sp > 0) {
        sp -= 1;
        int64_t node = tstack[sp];
        if (!aabb_hit(ox, oy, oz, ix, iy, iz, t_min, t_max, bd->t_bounds + 6 * node)) continue;
        int64_t cnt = bd->t_count[node];
        if (cnt > 0) {
            int64_t first = bd->t_left[node];
            for (int64_t k = 0; k < cnt; ++k) {
                int64_t inst = bd->t_order[first + k];
                if ((bd->i_mask[inst] & ray_mask) == 0) continue;
                double lo[3], ld[3];
                to_local(bd->i_inv + 12 * inst, ox, oy, oz, dx, dy, dz, lo, ld);
                if (blas_any(bd, bd->i_blas[inst], lo[0], lo[1], lo[2], ld[0], ld[1], ld[2], t_min, t_max) == 1)
                    return 1;
            }
        } else {
            tstack[sp] = bd->t_left[node];
            tstack[sp + 1] = bd->t_right[node];
            sp += 2;
        }
    }
    return 0;
}

/* ---- threading helper: split [0, n) into contiguous chunks like render_frame ---- */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void* ctx; int64_t lo, hi; } range_job;
static void* range_thread(void* p) { range_job* j = (range_job*)p; j->fn(j->ctx, j->lo, j->hi); return NULL; }

static void parallel_ranges(range_fn fn, void* ctx, int64_t n, int workers)
{
    if (workers <= 1 || n < 2) { fn(ctx, 0, n); return; }
    if (workers > n) workers = (int)n;
    pthread_t th[256];
    range_job jobs[256];
    if (workers > 256) workers = 256;
    for (int w = 0; w < workers; ++w) {
        /* np.linspace(0, n, workers+1, dtype=int64) */
        jobs[w].fn = fn; jobs[w].ctx = ctx;
        jobs[w].lo = (int64_t)((double)n * w / workers);
        jobs[w].hi = (int64_t)((double)n * (w + 1) / workers);
        pthread_create(&th[w], NULL, range_thread, &jobs[w]);
    }
    for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
}

/* accel.py:950-976 _closest_batch, out (n,5) = [t, inst, prim, u, v], out_n (n,3), stats (n,2) */
typedef struct {
    const orc_bundle* bd; const double *o, *d, *tmin, *tmax; uint64_t mask;
    double* out; double* out_n; int64_t* stats;
} closest_ctx;

static void closest_range(void* p, int64_t lo, int64_t hi)
{
    closest_ctx* c = (closest_ctx*)p;
    for (int64_t i = lo; i < hi; ++i) {
        orc_hit h;
        int st = tlas_closest(c->bd, c->o[3 * i], c->o[3 * i + 1], c->o[3 * i + 2],
                              c->d[3 * i], c->d[3 * i + 1], c->d[3 * i + 2], c->tmin[i], c->tmax[i], c->mask, &h);
        if (st == 0) {
            c->out[5 * i] = -1.0;
        } else {
            c->out[5 * i] = h.t; c->out[5 * i + 1] = (double)h.inst; c->out[5 * i + 2] = (double)h.prim;
            c->out[5 * i + 3] = h.u; c->out[5 * i + 4] = h.v;
            c->out_n[3 * i] = h.nx; c->out_n[3 * i + 1] = h.ny; c->out_n[3 * i + 2] = h.nz;
        }
        if (c->stats) { c->stats[2 * i] = h.tests; c->stats[2 * i + 1] = h.visits; }
    }
}

ORC_API int orc_closest_batch(const orc_bundle* bd, int64_t n, const double* o, const double* d,
                              const double* tmin, const double* tmax, uint64_t mask,
                              double* out, double* out_n, int64_t* stats, int workers)
{
    closest_ctx c = {bd, o, d, tmin, tmax, mask, out, out_n, stats};
    parallel_ranges(closest_range, &c, n, workers);
    return 0;
}

typedef struct {
    const orc_bundle* bd; const double *o, *d, *tmin, *tmax; uint64_t mask; uint8_t* out;
} any_ctx;

static void any_range(void* p, int64_t lo, int64_t hi)
{
    any_ctx* c = (any_ctx*)p;
    for (int64_t i = lo; i < hi; ++i)
        c->out[i] = (uint8_t)tlas_any(c->bd, c->o[3 * i], c->o[3 * i + 1], c->o[3 * i + 2],
                                      c->d[3 * i], c->d[3 * i + 1], c->d[3 * i + 2], c->tmin[i], c->tmax[i], c->mask);
}

ORC_API int orc_any_batch(const orc_bundle* bd, int64_t n, const double* o, const double* d,
                          const double* tmin, const double* tmax, uint64_t mask, uint8_t* out, int workers)
{
    any_ctx c = {bd, o, d, tmin, tmax, mask, out};
    parallel_ranges(any_range, &c, n, workers);
    return 0;
}

/* ======================================================================== */
/* Part A.4  RNG and sampling (sampling.py, camera.py)                      */
/* ======================================================================== */

#define PCG_MULT 6364136223846793005ULL
#define MIX_GAMMA 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z)   /* sampling.py:38-43 */
{
    z = z + MIX_GAMMA;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint32_t pcg_next(uint64_t* state, uint64_t inc)   /* sampling.py:46-54 */
{
    uint64_t old = *state;
    *state = old * PCG_MULT + inc;
    uint32_t xorshifted = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

static inline void stream_for(uint64_t seed, uint64_t pix, uint64_t s, uint64_t* state, uint64_t* inc)
{
    /* sampling.py:57-73 */
    uint64_t h = mix64(seed);
    h = mix64(h ^ pix);
    h = mix64(h ^ s);
    uint64_t initseq = mix64(h ^ 0xDA3E39CB94B95BDBULL);
    *inc = (initseq << 1) | 1ULL;
    *state = 0;
    pcg_next(state, *inc);
    *state += h;
    pcg_next(state, *inc);
}

static inline double uniform01(uint64_t* state, uint64_t inc)    /* sampling.py:76-79 */
{
    return (double)pcg_next(state, inc) * 0x1p-32;
}

ORC_API void orc_stream_for(uint64_t seed, uint64_t pix, uint64_t s, uint64_t* state, uint64_t* inc)
{
    stream_for(seed, pix, s, state, inc);
}

ORC_API void orc_uniforms(uint64_t seed, uint64_t pix, uint64_t s, int64_t n, double* out)
{
    uint64_t st, inc;
    stream_for(seed, pix, s, &st, &inc);
    for (int64_t i = 0; i < n; ++i) out[i] = uniform01(&st, inc);
}

static inline void cosine_dir(double x0, double x1, double* x, double* y, double* z)
{
    /* sampling.py:144-151 */
    double phi = 2.0 * M_PI * x0;
    double r = sqrt(x1);
    *x = cos(phi) * r;
    *z = sin(phi) * r;
    double q = 1.0 - r * r;
    *y = sqrt(q > 0.0 ? q : 0.0);
}

static inline void onb(double nx, double ny, double nz, double* t, double* b)
{
    /* sampling.py:175-186 */
    double s = copysign(1.0, nz);
    double a = -1.0 / (s + nz);
    double bb = nx * ny * a;
    t[0] = 1.0 + s * nx * nx * a;
    t[1] = s * bb;
    t[2] = -s * nx;
    b[0] = bb;
    b[1] = s + ny * ny * a;
    b[2] = -ny;
}

ORC_API void orc_cosine_dir(double x0, double x1, double* out3) { cosine_dir(x0, x1, out3, out3 + 1, out3 + 2); }
ORC_API void orc_onb(double nx, double ny, double nz, double* out6) { onb(nx, ny, nz, out6, out6 + 3); }

/* camera.py:81-97; cam = (origin3, right3, up3, forward3, distortion) */
static inline int primary_dir(const double* cam, double u, double v, double* d)
{
    double rx = cam[3], ry = cam[4], rz = cam[5], ux = cam[6], uy = cam[7], uz = cam[8];
    double fx = cam[9], fy = cam[10], fz = cam[11], dist = cam[12];
    double su = 2.0 * u - 1.0, sv = 1.0 - 2.0 * v;
    double px = rx * su + ux * sv, py = ry * su + uy * sv, pz = rz * su + uz * sv;
    double c = dist * (px * px + py * py + pz * pz);
    double denom = 1.0 + c;
    if (denom <= 0.0) { d[0] = d[1] = d[2] = 0.0; return 0; }
    double dx = fx + px / denom, dy = fy + py / denom, dz = fz + pz / denom;
    double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
    d[0] = dx * inv; d[1] = dy * inv; d[2] = dz * inv;
    return 1;
}

ORC_API int orc_primary_dir(const double* cam, double u, double v, double* d) { return primary_dir(cam, u, v, d); }

/* ======================================================================== */
/* Part A.5  integrators (integrators.py)                                   */
/* ======================================================================== */

typedef struct {
    const double* mat_color;     /* (M,3) */
    const double* mat_emissive;  /* (M,3) */
    const int64_t* inst_material;/* (I,) */
    const double *lv0, *lv1, *lv2, *ln, *lemis, *larea;  /* lights (L,3) / (L,) */
    int64_t n_lights;
    const double* sky;           /* 3 */
    const double* background;    /* 3 */
} orc_shade;

#define RAY_FAR 1e30
#define FULL_MASK 0xFFFFFFFFULL

static inline double geom_term(double px, double py, double pz, double npx, double npy, double npz,
                               double qx, double qy, double qz, double nqx, double nqy, double nqz)
{
    /* integrators.py:99-115 */
    double wx = qx - px, wy = qy - py, wz = qz - pz;
    double d2 = wx * wx + wy * wy + wz * wz;
    if (d2 <= 0.0) return 0.0;
    double inv = 1.0 / sqrt(d2);
    wx *= inv; wy *= inv; wz *= inv;
    double cos_p = npx * wx + npy * wy + npz * wz;
    double cos_q = -(nqx * wx + nqy * wy + nqz * wz);
    if (cos_p <= 0.0 || cos_q <= 0.0) return 0.0;
    return cos_p * cos_q / d2;
}

typedef struct {
    const orc_bundle* bd; const orc_shade* sh; const double* cam;
    int integ, max_depth, ao_count; double ao_length, normal_offset;
    int64_t width, height, spp, s0; uint64_t seed; int jitter;
    double* acc; int64_t* rays_per_worker; int64_t nworkers_slots;
    pthread_mutex_t* lock; int64_t* total_rays;
} render_ctx;

/* integrators.py:129-141 */
static void sample_eye(const render_ctx* c, double u, double v, double* rgb, int64_t* nr)
{
    double d[3];
    primary_dir(c->cam, u, v, d);
    orc_hit h;
    int st = tlas_closest(c->bd, c->cam[0], c->cam[1], c->cam[2], d[0], d[1], d[2], 0.0, RAY_FAR, FULL_MASK, &h);
    *nr = 1;
    if (st == 0) { rgb[0] = c->sh->background[0]; rgb[1] = c->sh->background[1]; rgb[2] = c->sh->background[2]; return; }
    int64_t m = c->sh->inst_material[h.inst];
    rgb[0] = c->sh->mat_color[3 * m]; rgb[1] = c->sh->mat_color[3 * m + 1]; rgb[2] = c->sh->mat_color[3 * m + 2];
}

/* integrators.py:144-179 */
static double sample_ao(const render_ctx* c, double u, double v, uint64_t* state, uint64_t inc, int64_t* nr)
{
    double d[3];
    primary_dir(c->cam, u, v, d);
    orc_hit h;
    int st = tlas_closest(c->bd, c->cam[0], c->cam[1], c->cam[2], d[0], d[1], d[2], 0.0, RAY_FAR, FULL_MASK, &h);
    *nr = 1;
    if (st == 0) return 1.0;
    double nx = h.nx, ny = h.ny, nz = h.nz;
    if (nx * d[0] + ny * d[1] + nz * d[2] > 0.0) { nx = -nx; ny = -ny; nz = -nz; }
    double px = c->cam[0] + d[0] * h.t + nx * c->normal_offset;
    double py = c->cam[1] + d[1] * h.t + ny * c->normal_offset;
    double pz = c->cam[2] + d[2] * h.t + nz * c->normal_offset;
    double t[3], b[3];
    onb(nx, ny, nz, t, b);
    int64_t occluded = 0;
    for (int i = 0; i < c->ao_count; ++i) {
        double x0 = uniform01(state, inc), x1 = uniform01(state, inc);
        double sx, sy, sz;
        cosine_dir(x0, x1, &sx, &sy, &sz);
        double wx = t[0] * sx + nx * sy + b[0] * sz;
        double wy = t[1] * sx + ny * sy + b[1] * sz;
        double wz = t[2] * sx + nz * sy + b[2] * sz;
        occluded += tlas_any(c->bd, px, py, pz, wx, wy, wz, 0.0, c->ao_length, FULL_MASK);
        *nr += 1;
    }
    return 1.0 - (double)occluded / (double)c->ao_count;
}

/* integrators.py:182-235 (nee=0) and 238-331 (nee=1) */
static void sample_pt(const render_ctx* c, int nee, double u, double v, uint64_t* state, uint64_t inc,
                      double* rgb, int64_t* nr)
{
    const orc_shade* sh = c->sh;
    double dd[3];
    primary_dir(c->cam, u, v, dd);
    double dx = dd[0], dy = dd[1], dz = dd[2];
    double ox = c->cam[0], oy = c->cam[1], oz = c->cam[2];
    double rr = 0, rg = 0, rb = 0, tr = 1, tg = 1, tb = 1;
    int64_t nrays = 0;
    double off = c->normal_offset;
    for (int depth = 0; depth < c->max_depth; ++depth) {
        orc_hit h;
        int st = tlas_closest(c->bd, ox, oy, oz, dx, dy, dz, 0.0, RAY_FAR, FULL_MASK, &h);
        nrays += 1;
        if (st == 0) { rr += tr * sh->sky[0]; rg += tg * sh->sky[1]; rb += tb * sh->sky[2]; break; }
        int64_t m = sh->inst_material[h.inst];
        double er = sh->mat_emissive[3 * m], eg = sh->mat_emissive[3 * m + 1], eb = sh->mat_emissive[3 * m + 2];
        if (er > 0.0 || eg > 0.0 || eb > 0.0) {
            if (!nee || depth == 0) { rr += tr * er; rg += tg * eg; rb += tb * eb; }
            break;
        }
        double nx = h.nx, ny = h.ny, nz = h.nz;
        if (nx * dx + ny * dy + nz * dz > 0.0) { nx = -nx; ny = -ny; nz = -nz; }
        double px = ox + dx * h.t, py = oy + dy * h.t, pz = oz + dz * h.t;
        if (nee) {
            double x0 = uniform01(state, inc), x1 = uniform01(state, inc), x2 = uniform01(state, inc);
            int64_t nl = sh->n_lights;
            int64_t li = (int64_t)(x0 * (double)nl);
            if (li > nl - 1) li = nl - 1;
            double s = sqrt(x1);
            double w0 = 1.0 - s, w1 = s * (1.0 - x2), w2 = s * x2;
            double qx = w0 * sh->lv0[3 * li] + w1 * sh->lv1[3 * li] + w2 * sh->lv2[3 * li];
            double qy = w0 * sh->lv0[3 * li + 1] + w1 * sh->lv1[3 * li + 1] + w2 * sh->lv2[3 * li + 1];
            double qz = w0 * sh->lv0[3 * li + 2] + w1 * sh->lv1[3 * li + 2] + w2 * sh->lv2[3 * li + 2];
            const double* lnrm = sh->ln + 3 * li;
            double g = geom_term(px, py, pz, nx, ny, nz, qx, qy, qz, lnrm[0], lnrm[1], lnrm[2]);
            if (g > 0.0) {
                double spx = px + nx * off, spy = py + ny * off, spz = pz + nz * off;
                double sqx = qx + lnrm[0] * off, sqy = qy + lnrm[1] * off, sqz = qz + lnrm[2] * off;
                int occ = tlas_any(c->bd, spx, spy, spz, sqx - spx, sqy - spy, sqz - spz, 0.0, 1.0 - 1e-3, FULL_MASK);
                nrays += 1;
                if (occ == 0) {
                    double pdf = (1.0 / (double)nl) * (1.0 / sh->larea[li]);
                    double scale = g / (M_PI * pdf);
                    rr += tr * sh->mat_color[3 * m] * sh->lemis[3 * li] * scale;
                    rg += tg * sh->mat_color[3 * m + 1] * sh->lemis[3 * li + 1] * scale;
                    rb += tb * sh->mat_color[3 * m + 2] * sh->lemis[3 * li + 2] * scale;
                }
            }
        }
        double x0 = uniform01(state, inc), x1 = uniform01(state, inc);
        double sx, sy, sz;
        cosine_dir(x0, x1, &sx, &sy, &sz);
        double t[3], b[3];
        onb(nx, ny, nz, t, b);
        dx = t[0] * sx + nx * sy + b[0] * sz;
        dy = t[1] * sx + ny * sy + b[1] * sz;
        dz = t[2] * sx + nz * sy + b[2] * sz;
        tr *= sh->mat_color[3 * m];
        tg *= sh->mat_color[3 * m + 1];
        tb *= sh->mat_color[3 * m + 2];
        ox = px + nx * off; oy = py + ny * off; oz = pz + nz * off;
    }
    rgb[0] = rr; rgb[1] = rg; rgb[2] = rb;
    *nr = nrays;
}

/* integrators.py:334-379 for pixels [lo, hi), samples [s0, s0+spp) */
static void render_range(void* p, int64_t lo, int64_t hi)
{
    render_ctx* c = (render_ctx*)p;
    int64_t total = 0;
    for (int64_t pix = lo; pix < hi; ++pix) {
        int64_t xi = pix % c->width, yi = pix / c->width;
        for (int64_t s = c->s0; s < c->s0 + c->spp; ++s) {
            uint64_t state, inc;
            stream_for(c->seed, (uint64_t)pix, (uint64_t)s, &state, &inc);
            double ju = 0.0, jv = 0.0;
            if (c->jitter) { ju = uniform01(&state, inc); jv = uniform01(&state, inc); }
            double u = ((double)xi + ju) / (double)c->width;
            double v = ((double)yi + jv) / (double)c->height;
            double rgb[3];
            int64_t nr = 0;
            if (c->integ == 0) sample_eye(c, u, v, rgb, &nr);
            else if (c->integ == 1) { double a = sample_ao(c, u, v, &state, inc, &nr); rgb[0] = rgb[1] = rgb[2] = a; }
            else sample_pt(c, c->integ == 3, u, v, &state, inc, rgb, &nr);
            c->acc[4 * pix] += rgb[0];
            c->acc[4 * pix + 1] += rgb[1];
            c->acc[4 * pix + 2] += rgb[2];
            c->acc[4 * pix + 3] += 1.0;
            total += nr;
        }
    }
    pthread_mutex_lock(c->lock);
    *c->total_rays += total;
    pthread_mutex_unlock(c->lock);
}

/*
 * integrators.py:426-473 render_frame core.  integ: 0 eye, 1 ao, 2 pt, 3 pt-nee.
 * acc is (H*W, 4) float64, accumulated in place (pixel rows top-down).
 * pix_lo/pix_hi restrict the pixel range (whole frame: 0, W*H).
 */
ORC_API int64_t orc_render(const orc_bundle* bd, const orc_shade* sh, const double* cam, int integ,
                           int max_depth, int ao_count, double ao_length, double normal_offset,
                           int64_t width, int64_t height, int64_t s0, int64_t spp, uint64_t seed, int jitter,
                           int64_t pix_lo, int64_t pix_hi, double* acc, int workers)
{
    pthread_mutex_t lock = PTHREAD_MUTEX_INITIALIZER;
    int64_t total = 0;
    render_ctx c;
    memset(&c, 0, sizeof c);
    c.bd = bd; c.sh = sh; c.cam = cam; c.integ = integ; c.max_depth = max_depth; c.ao_count = ao_count;
    c.ao_length = ao_length; c.normal_offset = normal_offset; c.width = width; c.height = height;
    c.spp = spp; c.s0 = s0; c.seed = seed; c.jitter = jitter; c.acc = acc; c.lock = &lock; c.total_rays = &total;
    if (workers <= 1 || pix_hi - pix_lo < 2) {
        render_range(&c, pix_lo, pix_hi);
    } else {
        /* offset ranges into [pix_lo, pix_hi) */
        int64_t n = pix_hi - pix_lo;
        int w = workers > 256 ? 256 : workers;
        if (w > n) w = (int)n;
        pthread_t th[256];
        range_job jobs[256];
        for (int k = 0; k < w; ++k) {
            jobs[k].fn = render_range; jobs[k].ctx = &c;
            jobs[k].lo = pix_lo + (int64_t)((double)n * k / w);
            jobs[k].hi = pix_lo + (int64_t)((double)n * (k + 1) / w);
            pthread_create(&th[k], NULL, range_thread, &jobs[k]);
        }
        for (int k = 0; k < w; ++k) pthread_join(th[k], NULL);
    }
    return total;
}

/* ======================================================================== */
/* Part B  CPU LBVH restatement (frozen choices)    */
/* ======================================================================== */

static inline uint32_t expand10(uint32_t v)
{
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

static inline uint64_t expand21(uint64_t v)
{
    v &= 0x1FFFFFull;
    v = (v | (v << 32)) & 0x001F00000000FFFFull;
    v = (v | (v << 16)) & 0x001F0000FF0000FFull;
    v = (v | (v << 8)) & 0x100F00F00F00F00Full;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

static inline float f32min(float a, float b) { return b < a ? b : a; }
static inline float f32max(float a, float b) { return b > a ? b : a; }

/* triangle AABB + centroid, fp32.  tri: (n, 9) world vertices */
static inline void tri_box(const float* t, float* lo, float* hi)
{
    for (int a = 0; a < 3; ++a) {
        lo[a] = f32min(f32min(t[a], t[3 + a]), t[6 + a]);
        hi[a] = f32max(f32max(t[a], t[3 + a]), t[6 + a]);
    }
}

/* quantise one centroid coordinate: q = (c - lo) * inv_ext * 2^b, clamped, truncated */
static inline uint32_t quantise(float c, float lo, float inv_ext, float scale, float qmax)
{
    volatile float d = c - lo;       /* separate fp32 sub, mul, mul: no contraction */
    volatile float e = d * inv_ext;
    float q = e * scale;
    q = f32max(q, 0.0f);
    q = f32min(q, qmax);
    return (uint32_t)q;
}

/* centroid bounds (lo3, hi3) and inv_ext (3) exactly as the GPU computes them */
ORC_API void orc_lbvh_bounds(int64_t n, const float* tris, float* cb6, float* inv_ext3)
{
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i) {
        float blo[3], bhi[3];
        tri_box(tris + 9 * i, blo, bhi);
        for (int a = 0; a < 3; ++a) {
            volatile float s = blo[a] + bhi[a];
            float c = 0.5f * s;
            lo[a] = f32min(lo[a], c);
            hi[a] = f32max(hi[a], c);
        }
    }
    for (int a = 0; a < 3; ++a) {
        cb6[a] = lo[a]; cb6[3 + a] = hi[a];
        volatile float ext = hi[a] - lo[a];
        inv_ext3[a] = ext > 0.0f ? 1.0f / ext : 0.0f;
    }
}

/* Morton keys (unsorted, key i belongs to triangle i) */
ORC_API void orc_lbvh_morton(int64_t n, const float* tris, int bits, const float* cb6, const float* inv_ext3,
                             uint64_t* keys)
{
    int b = bits == 63 ? 21 : 10;
    float scale = (float)(1u << b);
    float qmax = (float)((1u << b) - 1u);
    for (int64_t i = 0; i < n; ++i) {
        float blo[3], bhi[3];
        tri_box(tris + 9 * i, blo, bhi);
        uint32_t q[3];
        for (int a = 0; a < 3; ++a) {
            volatile float s = blo[a] + bhi[a];
            float c = 0.5f * s;
            q[a] = quantise(c, cb6[a], inv_ext3[a], scale, qmax);
        }
        if (b == 10)
            keys[i] = ((uint64_t)expand10(q[0]) << 2) | ((uint64_t)expand10(q[1]) << 1) | (uint64_t)expand10(q[2]);
        else
            keys[i] = (expand21(q[0]) << 2) | (expand21(q[1]) << 1) | expand21(q[2]);
    }
}

/* stable sort by (key, index): LSD radix on 16-bit digits, values = triangle ids */
ORC_API void orc_lbvh_sort(int64_t n, const uint64_t* keys_in, int bits, uint64_t* keys_out, uint32_t* order_out)
{
    uint64_t* ka = (uint64_t*)malloc((size_t)n * 8), *kb = (uint64_t*)malloc((size_t)n * 8);
    uint32_t* va = (uint32_t*)malloc((size_t)n * 4), *vb = (uint32_t*)malloc((size_t)n * 4);
    memcpy(ka, keys_in, (size_t)n * 8);
    for (int64_t i = 0; i < n; ++i) va[i] = (uint32_t)i;
    int passes = bits == 63 ? 4 : 2;
    int64_t* cnt = (int64_t*)malloc(65536 * sizeof(int64_t));
    for (int p = 0; p < passes; ++p) {
        memset(cnt, 0, 65536 * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) cnt[(ka[i] >> (16 * p)) & 0xFFFF]++;
        int64_t run = 0;
        for (int d = 0; d < 65536; ++d) { int64_t c = cnt[d]; cnt[d] = run; run += c; }
        for (int64_t i = 0; i < n; ++i) {
            int64_t pos = cnt[(ka[i] >> (16 * p)) & 0xFFFF]++;
            kb[pos] = ka[i]; vb[pos] = va[i];
        }
        uint64_t* tk = ka; ka = kb; kb = tk;
        uint32_t* tv = va; va = vb; vb = tv;
    }
    memcpy(keys_out, ka, (size_t)n * 8);
    memcpy(order_out, va, (size_t)n * 4);
    free(ka); free(kb); free(va); free(vb); free(cnt);
}

static inline int clz32(uint32_t x) { return x ? __builtin_clz(x) : 32; }
static inline int clz64(uint64_t x) { return x ? __builtin_clzll(x) : 64; }

/* Karras delta: keys in W-bit words, index fallback for equal keys */
static inline int karras_delta(const uint64_t* k, int64_t n, int64_t i, int64_t j, int wide)
{
    if (j < 0 || j > n - 1) return -1;
    uint64_t a = k[i], b = k[j];
    int W = wide ? 64 : 32;
    if (a != b) return wide ? clz64(a ^ b) : clz32((uint32_t)(a ^ b));
    return W + clz32((uint32_t)i ^ (uint32_t)j);
}

/*
 * Karras 2012 topology.  Internal nodes 0..n-2 (root 0), leaves n-1+i.
 * child: (n-1, 2) int32, >= 0 internal node, < 0 = ~leaf (leaf i -> -(i+1)).
 * parent: (2n-1) int32 over [internal..., leaves...]; root -> -1.
 */
ORC_API void orc_lbvh_karras(int64_t n, const uint64_t* keys, int bits, int32_t* child, int32_t* parent)
{
    int wide = bits == 63;
    parent[0] = -1;
    for (int64_t i = 0; i < n - 1; ++i) {
        int d = (karras_delta(keys, n, i, i + 1, wide) - karras_delta(keys, n, i, i - 1, wide)) >= 0 ? 1 : -1;
        int dmin = karras_delta(keys, n, i, i - d, wide);
        int64_t lmax = 2;
        while (karras_delta(keys, n, i, i + lmax * d, wide) > dmin) lmax *= 2;
        int64_t l = 0;
        for (int64_t t = lmax / 2; t >= 1; t /= 2)
            if (karras_delta(keys, n, i, i + (l + t) * d, wide) > dmin) l += t;
        int64_t j = i + l * d;
        int dnode = karras_delta(keys, n, i, j, wide);
        int64_t s = 0, t = l;
        do {
            t = (t + 1) >> 1;
            if (karras_delta(keys, n, i, i + (s + t) * d, wide) > dnode) s += t;
        } while (t > 1);
        int64_t gamma = i + s * d + (d < 0 ? d : 0);
        int64_t lo = i < j ? i : j, hi = i < j ? j : i;
        int32_t left = (lo == gamma) ? -(int32_t)(gamma + 1) : (int32_t)gamma;
        int32_t right = (hi == gamma + 1) ? -(int32_t)(gamma + 2) : (int32_t)(gamma + 1);
        child[2 * i] = left;
        child[2 * i + 1] = right;
        parent[left < 0 ? (n - 1) + (-left - 1) : left] = (int32_t)i;
        parent[right < 0 ? (n - 1) + (-right - 1) : right] = (int32_t)i;
    }
}

/*
 * Refit: child boxes per internal node, boxes (n-1, 12) = [lo_L, hi_L, lo_R, hi_R];
 * leaf i box = AABB of sorted triangle order[i]; heights (n-1) = 1 + max child height
 * (leaf height 0).  Returns tree height (root) which bounds the traversal stack.
 */
ORC_API int orc_lbvh_refit(int64_t n, const float* tris, const uint32_t* order, const int32_t* child,
                           float* boxes, int32_t* height, float* root6)
{
    if (n == 1) {
        float lo[3], hi[3];
        tri_box(tris + 9 * (int64_t)order[0], lo, hi);
        for (int a = 0; a < 3; ++a) { root6[a] = lo[a]; root6[3 + a] = hi[a]; }
        return 0;
    }
    /* post-order via explicit stack */
    float* nb = (float*)malloc((size_t)(n - 1) * 6 * sizeof(float));
    int64_t* stk = (int64_t*)malloc((size_t)(2 * n + 2) * sizeof(int64_t));
    uint8_t* seen = (uint8_t*)calloc((size_t)(n - 1), 1);
    int64_t sp = 0;
    stk[sp++] = 0;
    while (sp > 0) {
        int64_t i = stk[sp - 1];
        if (!seen[i]) {
            seen[i] = 1;
            for (int c = 1; c >= 0; --c) if (child[2 * i + c] >= 0) stk[sp++] = child[2 * i + c];
            continue;
        }
        sp--;
        int32_t h = 0;
        for (int c = 0; c < 2; ++c) {
            int32_t ch = child[2 * i + c];
            float lo[3], hi[3];
            int32_t chh;
            if (ch < 0) { tri_box(tris + 9 * (int64_t)order[-ch - 1], lo, hi); chh = 0; }
            else {
                for (int a = 0; a < 3; ++a) { lo[a] = nb[6 * ch + a]; hi[a] = nb[6 * ch + 3 + a]; }
                chh = height[ch];
            }
            for (int a = 0; a < 3; ++a) { boxes[12 * i + 6 * c + a] = lo[a]; boxes[12 * i + 6 * c + 3 + a] = hi[a]; }
            if (chh > h) h = chh;
        }
        height[i] = h + 1;
        for (int a = 0; a < 3; ++a) {
            nb[6 * i + a] = f32min(boxes[12 * i + a], boxes[12 * i + 6 + a]);
            nb[6 * i + 3 + a] = f32max(boxes[12 * i + 3 + a], boxes[12 * i + 9 + a]);
        }
    }
    for (int a = 0; a < 6; ++a) root6[a] = nb[a];
    int hroot = height[0];
    free(nb); free(stk); free(seen);
    return hroot;
}
