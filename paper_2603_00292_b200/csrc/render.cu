// render.cu -- K7 path-tracing megakernel and K8 wavefront path tracer
// (replace _render_chunk / _sample_eye / _sample_pt, integrators.py:129-235, 334-379).
//
// Both variants run the SAME per-bounce device code (shade_bounce) in fp32 in
// the reference's operation order, draw random numbers from the bit-exact
// per-(seed, pixel, sample) PCG32 stream (2 jitter draws, then 2 per bounce,
// integrators.py:345-351, 221-222) and accumulate each pixel in sample order,
// so mega and wavefront frames are bit-identical and independent of scheduling.
// World normals come per triangle from the host (reference-style);
// the ONB uses copysignf (signed-zero sensitive, sampling.py:175-186).  This
// TU must not be built with --use_fast_math.
#include <atomic>

#include "traverse.cuh"

namespace {

constexpr int MEGA_THREADS = 128;
#ifndef RT_TIMELINE
#define RT_TIMELINE 0           // diagnostic builds: per-warp start / end / SM / fetch count of the megakernel
#endif
#if RT_TIMELINE
#define RT_TIMELINE_WARPS 8192
__device__ unsigned long long g_timeline[4 * RT_TIMELINE_WARPS];
#endif
#ifndef RT_SMEM_STACK
#define RT_SMEM_STACK 0          // > 0: top entries of the megakernel's walk stack in shared memory
#endif
#ifndef MEGA_MIN_BLOCKS
#define MEGA_MIN_BLOCKS 7       // 72 registers: the 4-wide walk + PT shading without spills
#endif
constexpr int WF_THREADS = 256;

struct FrameConst {
    float cam[13];
    float sky[3];
    float bg[3];
    float offset;
    uint64_t seed;
    int width, height, jitter, integ, max_depth;
    int ao_count;
    float ao_length;
    int64_t pix_lo, npix;
    // work units: 8x4 pixel tiles (one per warp) when the range is whole rows
    int tiled, tiles_x;
    int band_stride, band_offset;   // interleaved tile-row bands (multi-GPU tile split)
    int64_t row0, row1, nunits;
    // tile-probe scheduling of single-sample tiled eye frames (see the megakernel)
    int probe_budget;              // walk steps of a probe ray; 0 = off (row-major tiles)
    unsigned epoch;                // this render's claim tag (claims[t] >= epoch: tile t taken)
    unsigned* claims;              // (tiles)
    unsigned long long* heavy_q;   // (tiles) (epoch << 32 | tile) of heavy tiles, in push order
    unsigned* probe_ctl;           // PC_WORDS control words (zeroed per render)
    unsigned* probe_hint;          // the scene's "last probed frame stopped" word
    // sample chunks of multi-sample frames (see the megakernel): 0 = one unit per tile
    int chunk;                     // samples per unit
    int nchunks;
    unsigned* chunk_done;          // (tiles) units of the tile finished, in sample order (zeroed per render)
    // eye frames of render_frame (rt_render_host): each pixel's sums from zero, written once
    // as float64 rows here (the fp32 accum is neither read nor written)
    double4* out64;
};

// unit k -> pixel; false for the padding lanes of partial edge tiles
__device__ __forceinline__ bool unit_pixel(const FrameConst& F, int64_t k, int64_t& pix) {
    if (!F.tiled) { pix = F.pix_lo + k; return true; }
    int64_t t = k >> 5;
    int l = (int)(k & 31);
    int64_t x = (t % F.tiles_x) * 8 + (l & 7);
    int64_t trow = (t / F.tiles_x) * F.band_stride + F.band_offset;
    int64_t y = F.row0 + trow * 4 + (l >> 3);
    pix = y * F.width + x;
    return x < F.width && y < F.row1;
}

struct PathState {
    float ox, oy, oz, dx, dy, dz;
    float tr, tg, tb, rr, rg, rb;
    uint64_t state, inc;
};

__device__ __forceinline__ void cosine_dir(float x0, float x1, float& x, float& y, float& z) {
    // sampling.py:144-151
    float phi = 2.0f * 3.14159265358979323846f * x0;
    float r = sqrtf(x1);
    float sp, cp;
    sincosf(phi, &sp, &cp);
    x = cp * r;
    z = sp * r;
    y = sqrtf(fmaxf(1.0f - r * r, 0.0f));
}

__device__ __forceinline__ void onb(float nx, float ny, float nz, float t[3], float b[3]) {
    // sampling.py:175-186 (copysign keeps the sign of a zero normal component)
    float s = copysignf(1.0f, nz);
    float a = -1.0f / (s + nz);
    float bb = nx * ny * a;
    t[0] = 1.0f + s * nx * nx * a;
    t[1] = s * bb;
    t[2] = -s * nx;
    b[0] = bb;
    b[1] = s + ny * ny * a;
    b[2] = -ny;
}

// integrators.py:345-351 + camera.py:81-97: stream, jitter, primary ray
__device__ __forceinline__ void start_path(const FrameConst& F, int64_t pix, int s, PathState& P,
                                           uint64_t hp) {
    rt_stream_from_pixel(hp, (uint64_t)s, P.state, P.inc);
    float ju = 0.0f, jv = 0.0f;
    if (F.jitter) {
        ju = rt_uniform(P.state, P.inc);
        jv = rt_uniform(P.state, P.inc);
    }
    int xi = (int)(pix % F.width), yi = (int)(pix / F.width);
    float u = ((float)xi + ju) / (float)F.width;
    float v = ((float)yi + jv) / (float)F.height;
    rt_primary_dir(F.cam, u, v, P.dx, P.dy, P.dz);
    P.ox = F.cam[0]; P.oy = F.cam[1]; P.oz = F.cam[2];
    P.tr = P.tg = P.tb = 1.0f;
    P.rr = P.rg = P.rb = 0.0f;
}

__device__ __forceinline__ void start_path(const FrameConst& F, int64_t pix, int s, PathState& P) {
    start_path(F, pix, s, P, rt_stream_pixel(F.seed, (uint64_t)pix));
}

// One closest-hit result applied to the path (integrators.py:129-141 eye,
// 198-235 pt).  Returns true if the path continues with a new ray.
template <bool SPH>
__device__ __forceinline__ bool shade_bounce(const FrameConst& F, const float4* __restrict__ attr,
                                             const float4* __restrict__ mat_color,
                                             const float4* __restrict__ mat_emis, const HitRec& h, PathState& P,
                                             const SphereView& sv) {
    if (F.integ == RT_INTEG_EYE) {
        if (h.id < 0) { P.rr = F.bg[0]; P.rg = F.bg[1]; P.rb = F.bg[2]; return false; }
        int m = __float_as_int(__ldg(attr + h.id).w);
        float4 c = __ldg(mat_color + m);
        P.rr = c.x; P.rg = c.y; P.rb = c.z;
        return false;
    }
    if (h.id < 0) {
        P.rr += P.tr * F.sky[0]; P.rg += P.tg * F.sky[1]; P.rb += P.tb * F.sky[2];
        return false;
    }
    float4 a = __ldg(attr + h.id);
    int m = __float_as_int(a.w);
    float4 e = __ldg(mat_emis + m);
    if (e.x > 0.0f || e.y > 0.0f || e.z > 0.0f) {
        P.rr += P.tr * e.x; P.rg += P.tg * e.y; P.rb += P.tb * e.z;
        return false;
    }
    float nx, ny, nz;
    hit_normal<SPH>(sv, h.id, a, P.ox, P.oy, P.oz, P.dx, P.dy, P.dz, h.t, nx, ny, nz);
    if (nx * P.dx + ny * P.dy + nz * P.dz > 0.0f) { nx = -nx; ny = -ny; nz = -nz; }
    float px = P.ox + P.dx * h.t, py = P.oy + P.dy * h.t, pz = P.oz + P.dz * h.t;
    float x0 = rt_uniform(P.state, P.inc);
    float x1 = rt_uniform(P.state, P.inc);
    float sx, sy, sz;
    cosine_dir(x0, x1, sx, sy, sz);
    float t[3], b[3];
    onb(nx, ny, nz, t, b);
    P.dx = t[0] * sx + nx * sy + b[0] * sz;
    P.dy = t[1] * sx + ny * sy + b[1] * sz;
    P.dz = t[2] * sx + nz * sy + b[2] * sz;
    float4 c = __ldg(mat_color + m);
    P.tr *= c.x; P.tg *= c.y; P.tb *= c.z;
    P.ox = px + nx * F.offset; P.oy = py + ny * F.offset; P.oz = pz + nz * F.offset;
    return true;
}

// integrators.py:99-115 _geom_term in fp32
__device__ __forceinline__ float geom_term(float px, float py, float pz, float npx, float npy, float npz, float qx,
                                           float qy, float qz, float nqx, float nqy, float nqz) {
    float wx = qx - px, wy = qy - py, wz = qz - pz;
    const float d2 = wx * wx + wy * wy + wz * wz;
    if (d2 <= 0.0f) return 0.0f;
    const float inv = 1.0f / sqrtf(d2);
    wx *= inv; wy *= inv; wz *= inv;
    const float cp = npx * wx + npy * wy + npz * wz;
    const float cq = -(nqx * wx + nqy * wy + nqz * wz);
    if (cp <= 0.0f || cq <= 0.0f) return 0.0f;
    return cp * cq / d2;
}

// integrators.py:144-179 _sample_ao: unoccluded fraction of the cosine lobe
template <bool SPH>
__device__ __forceinline__ float sample_ao(const FrameConst& F, const float4* __restrict__ bvh4, int root4,
                                           const float4* __restrict__ tris, const float4* __restrict__ attr,
                                           PathState& P, int2* stack, unsigned long long& rays, const SphereView& sv) {
    RayPre R;
    ray_setup(R, P.ox, P.oy, P.oz, P.dx, P.dy, P.dz, 0.0f);
    uint32_t nt, nv;
    const HitRec h = trace_ray4<false, SPH>(bvh4, root4, tris, R, 1e30f, RT_FULL, LocalStack{stack}, nt, nv, sv);
    ++rays;
    if (h.id < 0) return 1.0f;
    const float4 a = __ldg(attr + h.id);
    float nx, ny, nz;
    hit_normal<SPH>(sv, h.id, a, P.ox, P.oy, P.oz, P.dx, P.dy, P.dz, h.t, nx, ny, nz);
    if (nx * P.dx + ny * P.dy + nz * P.dz > 0.0f) { nx = -nx; ny = -ny; nz = -nz; }
    const float px = P.ox + P.dx * h.t + nx * F.offset;
    const float py = P.oy + P.dy * h.t + ny * F.offset;
    const float pz = P.oz + P.dz * h.t + nz * F.offset;
    float t[3], b[3];
    onb(nx, ny, nz, t, b);
    int occluded = 0;
    for (int k = 0; k < F.ao_count; ++k) {
        const float x0 = rt_uniform(P.state, P.inc), x1 = rt_uniform(P.state, P.inc);
        float sx, sy, sz;
        cosine_dir(x0, x1, sx, sy, sz);
        const float wx = t[0] * sx + nx * sy + b[0] * sz;
        const float wy = t[1] * sx + ny * sy + b[1] * sz;
        const float wz = t[2] * sx + nz * sy + b[2] * sz;
        RayPre S;
        ray_setup(S, px, py, pz, wx, wy, wz, 0.0f);
        occluded += trace_any4<SPH>(bvh4, root4, tris, S, F.ao_length, RT_FULL, reinterpret_cast<int*>(stack), sv) ? 1 : 0;
        ++rays;
    }
    return 1.0f - (float)occluded / (float)F.ao_count;
}

// integrators.py:238-331 _sample_ptnee: path tracing with one light connection per
// vertex (3 draws: light, then 2 for the area sample), emission counted only at depth 0
template <bool SPH>
__device__ __forceinline__ void sample_ptnee(const FrameConst& F, const float4* __restrict__ bvh4, int root4,
                                             const float4* __restrict__ tris, const float4* __restrict__ attr,
                                             const float4* __restrict__ mat_color, const float4* __restrict__ mat_emis,
                                             const float4* __restrict__ lights, int n_lights, PathState& P,
                                             int2* stack, unsigned long long& rays, const SphereView& sv) {
    for (int depth = 0; depth < F.max_depth; ++depth) {
        RayPre R;
        ray_setup(R, P.ox, P.oy, P.oz, P.dx, P.dy, P.dz, 0.0f);
        uint32_t nt, nv;
        const HitRec h = trace_ray4<false, SPH>(bvh4, root4, tris, R, 1e30f, RT_FULL, LocalStack{stack}, nt, nv, sv);
        ++rays;
        if (h.id < 0) {
            P.rr += P.tr * F.sky[0]; P.rg += P.tg * F.sky[1]; P.rb += P.tb * F.sky[2];
            return;
        }
        const float4 a = __ldg(attr + h.id);
        const int m = __float_as_int(a.w);
        const float4 e = __ldg(mat_emis + m);
        if (e.x > 0.0f || e.y > 0.0f || e.z > 0.0f) {
            if (depth == 0) { P.rr += P.tr * e.x; P.rg += P.tg * e.y; P.rb += P.tb * e.z; }
            return;
        }
        float nx, ny, nz;
        hit_normal<SPH>(sv, h.id, a, P.ox, P.oy, P.oz, P.dx, P.dy, P.dz, h.t, nx, ny, nz);
        if (nx * P.dx + ny * P.dy + nz * P.dz > 0.0f) { nx = -nx; ny = -ny; nz = -nz; }
        const float px = P.ox + P.dx * h.t, py = P.oy + P.dy * h.t, pz = P.oz + P.dz * h.t;
        const float4 c = __ldg(mat_color + m);
        // explicit light connection
        const float x0 = rt_uniform(P.state, P.inc), x1 = rt_uniform(P.state, P.inc),
                    x2 = rt_uniform(P.state, P.inc);
        int li = (int)(x0 * (float)n_lights);
        if (li > n_lights - 1) li = n_lights - 1;
        const float s = sqrtf(x1), w0 = 1.0f - s, w1 = s * (1.0f - x2), w2 = s * x2;
        const float4 l0 = __ldg(lights + 5 * li), l1 = __ldg(lights + 5 * li + 1), l2 = __ldg(lights + 5 * li + 2);
        const float4 ln = __ldg(lights + 5 * li + 3), le = __ldg(lights + 5 * li + 4);
        const float qx = w0 * l0.x + w1 * l1.x + w2 * l2.x;
        const float qy = w0 * l0.y + w1 * l1.y + w2 * l2.y;
        const float qz = w0 * l0.z + w1 * l1.z + w2 * l2.z;
        const float g = geom_term(px, py, pz, nx, ny, nz, qx, qy, qz, ln.x, ln.y, ln.z);
        if (g > 0.0f) {
            const float spx = px + nx * F.offset, spy = py + ny * F.offset, spz = pz + nz * F.offset;
            const float sqx = qx + ln.x * F.offset, sqy = qy + ln.y * F.offset, sqz = qz + ln.z * F.offset;
            RayPre S;
            ray_setup(S, spx, spy, spz, sqx - spx, sqy - spy, sqz - spz, 0.0f);
            const bool occ = trace_any4<SPH>(bvh4, root4, tris, S, 1.0f - 1e-3f, RT_FULL, reinterpret_cast<int*>(stack), sv);
            ++rays;
            if (!occ) {
                const float pdf = (1.0f / (float)n_lights) * (1.0f / l0.w);
                const float scale = g / (3.14159265358979323846f * pdf);
                P.rr += P.tr * c.x * le.x * scale;
                P.rg += P.tg * c.y * le.y * scale;
                P.rb += P.tb * c.z * le.z * scale;
            }
        }
        // diffuse bounce, as plain path tracing
        const float b0 = rt_uniform(P.state, P.inc), b1 = rt_uniform(P.state, P.inc);
        float sx, sy, sz;
        cosine_dir(b0, b1, sx, sy, sz);
        float t[3], b[3];
        onb(nx, ny, nz, t, b);
        P.dx = t[0] * sx + nx * sy + b[0] * sz;
        P.dy = t[1] * sx + ny * sy + b[1] * sz;
        P.dz = t[2] * sx + nz * sy + b[2] * sz;
        P.tr *= c.x; P.tg *= c.y; P.tb *= c.z;
        P.ox = px + nx * F.offset; P.oy = py + ny * F.offset; P.oz = pz + nz * F.offset;
    }
}

// ---- tile-probe scheduling (eye frames) ---------------------------------------
// A persistent frame ends when its last walk ends.  On a dense mesh a few primary walks
// (grazing rays along the silhouette: ~230 dependent node fetches + triangle tests against
// a median of 8) take ~0.2 ms alone, and in row-major order the last rows' long walks start
// when the work runs out.  So the megakernel first probes every 8x4 tile with one ray
// walked under a budget of walk steps (a separate instantiation of the walk: the budget
// exit is not in the rendering walk's loop); a tile whose probe runs out of budget is
// pushed on a heavy-tile queue, and every warp takes queued heavy tiles before row-major
// ones (whoever claims a tile first renders it).  On the config-2 sphere the probe (lane 12
// of the tile) flags every tile whose slowest ray needs >= 100 steps at a budget of 24 (8 %
// of the tiles, tools/diag_probe.py).  Only the schedule changes: each pixel is rendered
// once, by one lane, exactly as before (claims: one atomicMax of the render's epoch per
// tile).
#ifndef RT_PT_CHUNK
#ifndef RT_RENDER_PDL
#define RT_RENDER_PDL 1         // counters zeroed by a kernel, frame launched with programmatic dependent launch
#endif
#define RT_PT_CHUNK 8           // samples per work unit of multi-sample PT / AO frames (0: whole tiles)
#endif
#ifndef RT_PROBE_BUDGET
#define RT_PROBE_BUDGET 24      // walk steps; the RT_PROBE_BUDGET env overrides (0: no probe)
#endif
#ifndef RT_PROBE_CAP_DIV
#define RT_PROBE_CAP_DIV 8      // heavy queue cap: tiles / 8
#endif
constexpr int PROBE_LANE = 12;  // (x 4, y 1) of the 8x4 tile
// tiles per probe batch (lanes 0..15 probe): the first wave, one batch per warp, covers a
// 1080p frame (4050 batches for 4144 warps) but only a quarter of a 4K one, so a uniformly
// costly 4K scene pays for 66K probe walks before the stop rule can see it
constexpr int PROBE_BATCH = 16;
// probe control words, one per 128-B line of F.probe_ctl
constexpr int PC_TAKEN = 0, PC_HEAD = 32, PC_TAIL = 64, PC_DONE = 96, PC_STOP = 128, PC_LIMIT = 160, PC_MODE = 192,
              PC_QTAG = 193, PC_ZERO = 224;
// persistent across frames (not zeroed): the last complete heavy-tile queue (length, tag,
// valid) and the epoch of the last frame
constexpr int PC_QLEN = 224, PC_QEPOCH = 225, PC_QVALID = 226, PC_EPOCH = 227, PC_WORDS = 256;
// frame modes (PC_MODE): row-major, probed (probe batches + heavy queue), replay (the heavy
// queue of the scene's last complete probe, no probe walks)
constexpr unsigned PM_ROW = 0, PM_PROBE = 1, PM_REPLAY = 2;
// A scene whose last probed frame stopped probing (uniformly costly: the 10M soup) renders its
// next frames row-major without probes, re-probing every RT_PROBE_REPROBE-th frame
#ifndef RT_PROBE_REPROBE
#define RT_PROBE_REPROBE 8
#endif
#ifndef RT_PROBE_REPLAY
#define RT_PROBE_REPLAY 1       // replay the last complete heavy-tile queue of the same scene
#endif
struct ProbeBudget {
    int it, budget;
    __device__ __forceinline__ bool tick() { return ++it > budget; }
};
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
    return *reinterpret_cast<const volatile unsigned*>(p);
}
// pop a heavy tile (lane 0): -1 when none is queued.  The queue head only moves by
// atomicAdd (a CAS loop livelocks under thousands of polling warps); a ticket taken past
// the producers' reservations waits for its slot to be filled, or gives up once every
// probe batch is complete (completion counts tiles: it reaches `ntiles_b`, the tile count
// rounded up to whole batches, exactly) and the final reservation count is at or below the
// ticket.  The control words (F.probe_ctl) sit on their own 128-B lines, away from the
// frame's work counter: a store into the line of the work counter's atomics, once per warp,
// was measured to double the frame.
__device__ __forceinline__ int64_t heavy_pop(const FrameConst& F, unsigned* pc, unsigned ntiles_b) {
    if (ld_volatile_u32(pc + PC_HEAD) >= ld_volatile_u32(pc + PC_TAIL)) return -1;
    const unsigned h = atomicAdd(pc + PC_HEAD, 1u);
    while (true) {
        const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(F.heavy_q + h);
        if ((unsigned)(e >> 32) == ld_volatile_u32(pc + PC_QTAG)) return (int64_t)(e & 0xFFFFFFFFull);
        unsigned done;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(done) : "l"(pc + PC_DONE) : "memory");
        if (done >= ntiles_b && h >= ld_volatile_u32(pc + PC_TAIL)) return -1;
    }
}

// Lane 0 of a probing warp: take the next probe batch (its first tile; >= ntiles when none
// is left) and decide whether it is walked.  When more than 1/8 of the probed tiles (after
// the first 4096) or tiles / 8 in all came out heavy, the scene is uniformly costly (no tail
// to fix: the 10M soup flags 31 %) and probing stops: the remaining batches are taken and
// completed without walks (the completion count must reach every batch: heavy_pop's
// termination test), and the first tile no walk can have touched is published in PC_LIMIT
// (+ 1, so 0 means "not stopped"): row-major fetches claim only the tiles below it.
// Batches are taken by acq_rel adds and the stopping warp reads the batch counter by one
// after its stop store, so a batch at or above the limit is always taken after the stop is
// visible to its prober.
__device__ __forceinline__ unsigned probe_take(const FrameConst& F, unsigned* pc, int64_t ntiles, unsigned& stop) {
    unsigned pb;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(pb) : "l"(pc + PC_TAKEN), "r"(PROBE_BATCH)
                 : "memory");
    const unsigned nh = ld_volatile_u32(pc + PC_TAIL);
    const bool seen_stop = ld_volatile_u32(pc + PC_STOP) != 0;
    stop = seen_stop || nh >= (unsigned)(ntiles / RT_PROBE_CAP_DIV) || (pb >= 4096u && nh * RT_PROBE_CAP_DIV > pb);
    if (stop && !seen_stop) {
        *reinterpret_cast<volatile unsigned*>(pc + PC_STOP) = 1u;
        *reinterpret_cast<volatile unsigned*>(F.probe_hint) = 1u;   // the scene's next frames skip the probe
        unsigned lim;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 0;" : "=r"(lim) : "l"(pc + PC_TAKEN) : "memory");
        atomicMax(pc + PC_LIMIT, lim + 1u);
    }
    return pb;
}

// Lane 0 of a rendering warp in a probed frame: the first unit of its next tile, -1 to fetch
// again (the tile was taken by someone else), >= nunits when the frame is done.  Queued heavy
// tiles come first (the queue is polled until it is drained after every probe batch
// completed, or abandoned when probing stopped early: its tiles are unclaimed and go back to
// row-major order, which L2 rewards on such scenes), then row-major tiles, each claimed by
// one atomicMax of the render's epoch (tiles past the probe's limit need no claim).
// qopen / limit: this warp's shared-memory copies (see the kernel).
__device__ __forceinline__ long long probed_next_tile(const FrameConst& F, unsigned* counter, unsigned* pc,
                                                      int64_t ntiles, unsigned& qopen, unsigned& limit) {
    if (qopen) {
        const unsigned ntiles_b = (unsigned)((ntiles + PROBE_BATCH - 1) / PROBE_BATCH * PROBE_BATCH);
        const unsigned lim = ld_volatile_u32(pc + PC_LIMIT);
        if (lim) {
            limit = lim;
            qopen = 0u;
        } else {
            const int64_t ht = heavy_pop(F, pc, ntiles_b);
            if (ht >= 0) return atomicMax(F.claims + ht, F.epoch) < F.epoch ? ht * 32 : -1;
            if (ld_volatile_u32(pc + PC_DONE) >= ntiles_b && ld_volatile_u32(pc + PC_HEAD) >= ld_volatile_u32(pc + PC_TAIL))
                qopen = 0u;
        }
    }
    const long long b = atomicAdd(counter, 32u);
    if (b < F.nunits && (limit == 0u || (b >> 5) + 1 < (long long)limit) &&
        atomicMax(F.claims + (b >> 5), F.epoch) >= F.epoch)
        return -1;
    return b;
}

// ---- K7: megakernel --------------------------------------------------------
// the megakernel's work counters and probe control words, zeroed by a kernel launched with
// programmatic dependent launch (it and the megakernel queue behind the previous kernel --
// e.g. the LBVH build's last -- without two memset nodes and their launch gaps)
// It also sets this eye frame's mode (PC_MODE).  Row-major when the scene's last probed
// frame stopped probing (the hint); a replay of the last complete heavy-tile queue when the
// previous probe-capable frame was of the same scene and tile geometry (replay_ok) and its
// queue is complete (a probe that ran to the end, or a replay of one); else a probed frame,
// which clears the hint (its own stop sets it again).  Every RT_PROBE_REPROBE-th frame
// probes.  A replay frame starts with every probe batch counted done and the old queue's
// length and tag (its tiles are claimed with this frame's epoch as usual).
__global__ void render_ctl_zero_kernel(unsigned* __restrict__ counter, unsigned* __restrict__ pc,
                                       unsigned* __restrict__ hint, unsigned epoch, int replay_ok,
                                       unsigned ntiles_b) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // the previous kernel (the BVH, a frame) is done
    __shared__ unsigned s_mode, s_qlen, s_qtag;
    const int t = threadIdx.x;
    if (t < 64) counter[t] = 0u;
    if (!pc) return;
    if (t == 0) {
        const unsigned pm = pc[PC_MODE];
        if (pm == PM_PROBE && pc[PC_STOP] == 0u) {         // the previous frame's complete queue
            pc[PC_QLEN] = pc[PC_TAIL];
            pc[PC_QEPOCH] = pc[PC_EPOCH];
            pc[PC_QVALID] = 1u;
        } else if (pm != PM_REPLAY) {
            pc[PC_QVALID] = 0u;
        }
        const bool reprobe = epoch % RT_PROBE_REPROBE == 0u;
        unsigned mode;
        if (*hint != 0u && !reprobe) mode = PM_ROW;
        else if (replay_ok && pc[PC_QVALID] && !reprobe) mode = PM_REPLAY;
        else {
            mode = PM_PROBE;
            *hint = 0u;
        }
        pc[PC_EPOCH] = epoch;
        s_mode = mode;
        s_qlen = pc[PC_QLEN];
        s_qtag = mode == PM_REPLAY ? pc[PC_QEPOCH] : epoch;
    }
    __syncthreads();
    if (t < PC_ZERO) {
        unsigned v = 0u;
        if (t == PC_MODE) v = s_mode;
        else if (t == PC_QTAG) v = s_qtag;
        else if (s_mode == PM_REPLAY && t == PC_TAIL) v = s_qlen;
        else if (s_mode == PM_REPLAY && t == PC_DONE) v = ntiles_b;
        pc[t] = v;
    }
}

// float64 copy of fp32 sums (render_frame's readback of every frame but the eye frames)
__global__ void widen_kernel(const float4* __restrict__ acc, double4* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = __ldcs(acc + i);
        out[i] = make_double4(a.x, a.y, a.z, a.w);
    }
}

// Persistent warps fetch 32 pixels at a time; each lane renders samples
// [s0, s1) of its pixel in order and adds the sums to accum once.
// OUT64: sums from zero written as float64 rows to F.out64 (rt_render_host, eye frames)
template <int INTEG, bool SPH, bool OUT64 = false>
__global__ void __launch_bounds__(MEGA_THREADS, MEGA_MIN_BLOCKS) pt_megakernel(
    const FrameConst F, int s0, int s1, const float4* __restrict__ nodes, const float4* __restrict__ bvh4,
    const float4* __restrict__ tris, const float4* __restrict__ attr, const float4* __restrict__ mat_color,
    const float4* __restrict__ mat_emis, const float4* __restrict__ lights, int n_lights,
    float4* __restrict__ accum, unsigned int* counter, unsigned long long* ray_total, int* err,
    const SphereView sv) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // zeroed counters (and the BVH) first
    const int height = __float_as_int(__ldg(nodes + 3).z);
    const int root4 = __float_as_int(__ldg(nodes + 3).w);
    if (height + 1 > RT_STACK) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(err, RT_EDEPTH);
        return;
    }
    int2 stack[RT_STACK4];
#if RT_SMEM_STACK
    // PT / eye walks: the top RT_SMEM_STACK entries in shared memory, the rest local
    __shared__ int2 s_stack[RT_SMEM_STACK * MEGA_THREADS];
    const SmemStack<RT_SMEM_STACK, MEGA_THREADS> walk_stack{s_stack + threadIdx.x, stack};
#else
    const LocalStack walk_stack{stack};
#endif
    const int lane = threadIdx.x & 31;
    unsigned long long rays = 0;
    const int max_depth = INTEG == RT_INTEG_EYE ? 1 : F.max_depth;
#if RT_TIMELINE
    unsigned long long t_start, t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    unsigned n_fetch = 0;
#endif
    unsigned* const pc = F.probe_ctl;
    const unsigned pmode = INTEG == RT_INTEG_EYE && F.probe_budget > 0 ? __ldcg(pc + PC_MODE) : PM_ROW;
    const bool probe_on = pmode != PM_ROW;
    const int64_t ntiles = F.nunits >> 5;
    // per-warp fetch state of the probed schedule, kept out of registers (the walk's loop is
    // register-bound): the heavy queue is still worth polling; the first unprobed tile + 1
    // once probing has stopped (0: not known)
    __shared__ unsigned s_qopen[MEGA_THREADS / 32], s_limit[MEGA_THREADS / 32];
    if (lane == 0) {
        s_qopen[threadIdx.x >> 5] = 1u;
        s_limit[threadIdx.x >> 5] = 0u;
    }
    __syncwarp();
    // warps beyond the batch count start on row-major work (no pile-up on the batch counter)
    bool probing = pmode == PM_PROBE &&
                   (int64_t)(blockIdx.x * (MEGA_THREADS / 32) + (threadIdx.x >> 5)) < (ntiles + PROBE_BATCH - 1) / PROBE_BATCH;
    while (true) {
        int64_t base;
        int cs0 = s0, cs1 = s1;                     // this unit's sample window
        int64_t ctile = -1;                         // chunked frames: the unit's tile
        if (F.nchunks > 1) {
            // sample-chunk units, chunk-major: unit u = (chunk u / tiles, tile u % tiles).  A
            // tile's chunk c starts only after its chunk c - 1 has finished (chunk_done), so
            // every pixel still accumulates its samples in order; one sweep apart, the wait is
            // all but never taken.  The frame's tail shrinks from one tile x all samples to one
            // tile x one chunk.
            unsigned u = 0;
            if (lane == 0) u = atomicAdd(counter, 1u);
            u = __shfl_sync(RT_FULL, u, 0);
            if ((int64_t)u >= ntiles * F.nchunks) break;
            const int c = (int)(u / ntiles);
            ctile = (int64_t)u - (int64_t)c * ntiles;
            cs0 = s0 + c * F.chunk;
            cs1 = min(s1, cs0 + F.chunk);
            if (c > 0 && lane == 0) {
                while (ld_volatile_u32(F.chunk_done + ctile) < (unsigned)c) __nanosleep(256);
            }
            __syncwarp();                           // (the sums are then read from L2, below)
            base = ctile * 32;
        } else if (!probe_on) {
            unsigned b = 0;
            if (lane == 0) b = atomicAdd(counter, 32u);
            b = __shfl_sync(RT_FULL, b, 0);
            if ((int64_t)b >= F.nunits) break;
            base = b;
        } else if (probing) {
            // one probe batch: PROBE_BATCH tiles, one budgeted walk each (lanes < PROBE_BATCH),
            // the heavy ones queued
            unsigned pb = 0, stop = 0;
            if (lane == 0) pb = probe_take(F, pc, ntiles, stop);
            pb = __shfl_sync(RT_FULL, pb, 0);
            stop = __shfl_sync(RT_FULL, stop, 0);
            if ((int64_t)pb >= ntiles) {
                probing = false;
                continue;
            }
            const int64_t t = (int64_t)pb + lane;
            bool heavy = false;
            int64_t ppix;
            if (!stop && lane < PROBE_BATCH && t < ntiles && unit_pixel(F, t * 32 + PROBE_LANE, ppix)) {
                PathState P;
                start_path(F, ppix, s0, P);
                RayPre R;
                ray_setup(R, P.ox, P.oy, P.oz, P.dx, P.dy, P.dz, 0.0f);
                uint32_t nt, nv;
                ProbeBudget y{0, F.probe_budget};
                heavy = trace_ray4_y<false, SPH>(bvh4, root4, tris, R, 1e30f, RT_FULL, walk_stack, nt, nv, sv, y).id ==
                        RT_YIELDED;
            }
            if (heavy) {
                const unsigned slot = atomicAdd(pc + PC_TAIL, 1u);
                *reinterpret_cast<volatile unsigned long long*>(F.heavy_q + slot) =
                    ((unsigned long long)F.epoch << 32) | (unsigned long long)t;
            }
            __syncwarp();
            // the batch's queue slots before its completion count (a release reduction: a full
            // fence here would also invalidate the SM's L1, which the walks live in)
            if (lane == 0)
                asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(pc + PC_DONE), "r"(PROBE_BATCH) : "memory");
            continue;
        } else {
            long long b = 0;
            if (lane == 0) b = probed_next_tile(F, counter, pc, ntiles, s_qopen[threadIdx.x >> 5], s_limit[threadIdx.x >> 5]);
            b = __shfl_sync(RT_FULL, b, 0);
            if (b >= F.nunits) break;
            if (b < 0) continue;                         // taken by someone else: fetch again
            base = b;
        }
#if RT_TIMELINE
        ++n_fetch;
#endif
        int64_t i = base + lane;
        int64_t pix;
        if (i < F.nunits && unit_pixel(F, i, pix)) {
            // accumulate sample by sample into the running sums, exactly like
            // the wavefront's per-wave accumulate, so both are bit-identical
            // a chunked unit reads the sums its tile's previous chunk left in L2 (released
            // before its chunk_done count; a full fence here would also drop the SM's L1)
            float4 a = OUT64 ? make_float4(0.f, 0.f, 0.f, 0.f) : ctile >= 0 ? __ldcg(accum + pix) : accum[pix];
            const uint64_t hp = rt_stream_pixel(F.seed, (uint64_t)pix);   // per pixel, not per sample
            for (int s = cs0; s < cs1; ++s) {
                PathState P;
                start_path(F, pix, s, P, hp);
                if constexpr (INTEG == RT_INTEG_AO) {
                    const float v = sample_ao<SPH>(F, bvh4, root4, tris, attr, P, stack, rays, sv);
                    P.rr = P.rg = P.rb = v;
                } else if constexpr (INTEG == RT_INTEG_PTNEE) {
                    sample_ptnee<SPH>(F, bvh4, root4, tris, attr, mat_color, mat_emis, lights, n_lights, P, stack, rays, sv);
                } else {
                    for (int depth = 0; depth < max_depth; ++depth) {
                        RayPre R;
                        ray_setup(R, P.ox, P.oy, P.oz, P.dx, P.dy, P.dz, 0.0f);
                        uint32_t nt, nv;
                        HitRec h = trace_ray4<false, SPH>(bvh4, root4, tris, R, 1e30f, RT_FULL, walk_stack, nt, nv, sv);
                        ++rays;
                        if (!shade_bounce<SPH>(F, attr, mat_color, mat_emis, h, P, sv)) break;
                    }
                }
                a.x += P.rr; a.y += P.rg; a.z += P.rb; a.w += 1.0f;
            }
            if constexpr (OUT64)
                F.out64[pix] = make_double4(a.x, a.y, a.z, a.w);
            else
                accum[pix] = a;
        }
        if (ctile >= 0) {
            __syncwarp();                           // every lane's sums, then one release by lane 0
            if (lane == 0)
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(F.chunk_done + ctile) : "memory");
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rays += __shfl_xor_sync(RT_FULL, rays, off);
    if (lane == 0 && rays) atomicAdd(ray_total, rays);
#if RT_TIMELINE
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    const unsigned w = blockIdx.x * (MEGA_THREADS / 32) + (threadIdx.x >> 5);
    if (lane == 0 && w < RT_TIMELINE_WARPS) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_timeline[4 * w] = t_start;
        g_timeline[4 * w + 1] = t_end;
        g_timeline[4 * w + 2] = smid;
        g_timeline[4 * w + 3] = n_fetch;
    }
#endif
}

// ---- K8: wavefront ----------------------------------------------------------
struct Wave {
    float4* ray;      // (npix, 2)  o+tmin, d+tmax   (trace layout)
    float4* thr;      // (npix)     throughput rgb
    float4* rad;      // (npix)     radiance rgb
    uint2* rng;       // (npix, 2)  state, inc
    float4* hit;      // (npix)
    int64_t* pix;     // (nunits)   pixel of each path slot, -1 for padding
    int* queue[2];    // ping-pong path-index queues
    unsigned int* count;   // [depth] live paths per depth (max_depth + 1)
};

__global__ void __launch_bounds__(WF_THREADS) wf_raygen(const FrameConst F, const int* __restrict__ d_sample,
                                                         Wave W) {
    const int s = *d_sample;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F.nunits; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t pix;
        bool ok = unit_pixel(F, i, pix);
        W.pix[i] = ok ? pix : -1;
        W.rad[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!ok) continue;
        PathState P;
        start_path(F, pix, s, P);
        W.ray[2 * i] = make_float4(P.ox, P.oy, P.oz, 0.0f);
        W.ray[2 * i + 1] = make_float4(P.dx, P.dy, P.dz, 1e30f);
        W.thr[i] = make_float4(1.f, 1.f, 1.f, 0.f);
        W.rng[2 * i] = make_uint2((unsigned)P.state, (unsigned)(P.state >> 32));
        W.rng[2 * i + 1] = make_uint2((unsigned)P.inc, (unsigned)(P.inc >> 32));
    }
    if (blockIdx.x == 0 && threadIdx.x <= F.max_depth) W.count[threadIdx.x] = threadIdx.x == 0 ? (unsigned)F.nunits : 0u;
}

// extend: closest hit for every queued path (depth 0: identity queue)
template <bool SPH>
__global__ void __launch_bounds__(128, 8) wf_extend(const float4* __restrict__ nodes, const float4* __restrict__ bvh4,
                                                    const float4* __restrict__ tris, Wave W, int depth,
                                                    unsigned int* counter, int* err, const SphereView sv) {
    const int height = __float_as_int(__ldg(nodes + 3).z);
    const int root4 = __float_as_int(__ldg(nodes + 3).w);
    if (height + 1 > RT_STACK) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(err, RT_EDEPTH);
        return;
    }
    int2 stack[RT_STACK4];
    const unsigned n = W.count[depth];
    const int* q = depth == 0 ? nullptr : W.queue[depth & 1];
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(counter + depth, 32u);
        base = __shfl_sync(RT_FULL, base, 0);
        if (base >= n) break;
        unsigned k = base + lane;
        if (k < n) {
            int i = q ? q[k] : (int)k;
            if (q || W.pix[i] >= 0) {
            float4 a = W.ray[2 * i], b = W.ray[2 * i + 1];
            RayPre R;
            ray_setup(R, a.x, a.y, a.z, b.x, b.y, b.z, a.w);
            uint32_t nt, nv;
            HitRec h = trace_ray4<false, SPH>(bvh4, root4, tris, R, b.w, RT_FULL, LocalStack{stack}, nt, nv, sv);
            W.hit[i] = make_float4(h.t, __int_as_float(h.id), h.u, h.v);
            }
        }
    }
}

// shade: apply the hit, bounce, append survivors to the next queue with one
// atomicAdd per warp (ballot + popc)
template <bool SPH>
__global__ void __launch_bounds__(WF_THREADS) wf_shade(const FrameConst F, const float4* __restrict__ attr,
                                                        const float4* __restrict__ mat_color,
                                                        const float4* __restrict__ mat_emis, Wave W, int depth,
                                                        const SphereView sv) {
    const unsigned n = W.count[depth];
    const int* q = depth == 0 ? nullptr : W.queue[depth & 1];
    int* qn = W.queue[(depth + 1) & 1];
    const bool last = depth + 1 >= (F.integ == RT_INTEG_EYE ? 1 : F.max_depth);
    const int lane = threadIdx.x & 31;
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned k0 = blockIdx.x * blockDim.x; k0 < n; k0 += stride) {
        unsigned k = k0 + threadIdx.x;
        bool alive = false;
        int i = -1;
        if (k < n && (q || W.pix[k] >= 0)) {
            i = q ? q[k] : (int)k;
            float4 h4 = W.hit[i];
            HitRec h;
            h.t = h4.x; h.id = __float_as_int(h4.y); h.u = h4.z; h.v = h4.w;
            float4 a = W.ray[2 * i], b = W.ray[2 * i + 1], tp = W.thr[i], rd = W.rad[i];
            uint2 s0 = W.rng[2 * i], s1 = W.rng[2 * i + 1];
            PathState P;
            P.ox = a.x; P.oy = a.y; P.oz = a.z; P.dx = b.x; P.dy = b.y; P.dz = b.z;
            P.tr = tp.x; P.tg = tp.y; P.tb = tp.z; P.rr = rd.x; P.rg = rd.y; P.rb = rd.z;
            P.state = ((uint64_t)s0.y << 32) | s0.x;
            P.inc = ((uint64_t)s1.y << 32) | s1.x;
            bool cont = shade_bounce<SPH>(F, attr, mat_color, mat_emis, h, P, sv);
            W.rad[i] = make_float4(P.rr, P.rg, P.rb, 0.f);
            if (cont && !last) {
                alive = true;
                W.ray[2 * i] = make_float4(P.ox, P.oy, P.oz, 0.0f);
                W.ray[2 * i + 1] = make_float4(P.dx, P.dy, P.dz, 1e30f);
                W.thr[i] = make_float4(P.tr, P.tg, P.tb, 0.f);
                W.rng[2 * i] = make_uint2((unsigned)P.state, (unsigned)(P.state >> 32));
            }
        }
        unsigned ballot = __ballot_sync(RT_FULL, alive);
        if (ballot) {
            unsigned slot = 0;
            if (lane == 0) slot = atomicAdd(W.count + depth + 1, __popc(ballot));
            slot = __shfl_sync(RT_FULL, slot, 0);
            if (alive) qn[slot + __popc(ballot & ((1u << lane) - 1u))] = i;
        }
    }
}

__global__ void __launch_bounds__(WF_THREADS) wf_accumulate(const FrameConst F, Wave W, float4* __restrict__ accum,
                                                             int* d_sample, unsigned int* counter,
                                                             unsigned long long* ray_total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F.nunits; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t pix = W.pix[i];
        if (pix < 0) continue;
        float4 r = W.rad[i];
        float4 a = accum[pix];
        a.x += r.x; a.y += r.y; a.z += r.z; a.w += 1.0f;
        accum[pix] = a;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // closest-hit queries: every real pixel at depth 0 (count[0] also holds the
        // padding lanes of partial edge tiles) + the live paths of later depths
        unsigned long long total = (unsigned long long)F.npix;
        int md = F.integ == RT_INTEG_EYE ? 1 : F.max_depth;
        for (int d = 1; d < md; ++d) total += W.count[d];
        *ray_total += total;
        *d_sample += 1;
        for (int d = 0; d <= md; ++d) counter[d] = 0;
    }
}

// scene_io.py:349-355 resolve: mean = sum / n, clamp to [0, 1], optional ^(1/2.2),
// round(255 v) half-to-even (np.round), in float64 from the fp32 running sums
__global__ void resolve_kernel(const float4* __restrict__ accum, int64_t npix, int gamma, uint8_t* __restrict__ rgb,
                               int* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = accum[i];
        if (!(a.w > 0.0f)) {
            atomicExch(err, RT_EINVAL);
            continue;
        }
        const double n = a.w;
        const double c[3] = {a.x / n, a.y / n, a.z / n};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double v = c[k] < 0.0 ? 0.0 : (c[k] > 1.0 ? 1.0 : c[k]);
            if (gamma) v = pow(v, 1.0 / 2.2);
            rgb[3 * i + k] = (uint8_t)rint(255.0 * v);
        }
    }
}

__global__ void raygen_kernel(const FrameConst F, int s, float4* __restrict__ rays) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F.npix; i += (int64_t)gridDim.x * blockDim.x) {
        PathState P;
        start_path(F, F.pix_lo + i, s, P);
        rays[2 * i] = make_float4(P.ox, P.oy, P.oz, 0.0f);
        rays[2 * i + 1] = make_float4(P.dx, P.dy, P.dz, 1e30f);
    }
}

FrameConst make_frame(const rt_render_params* p) {
    FrameConst F;
    for (int k = 0; k < 13; ++k) F.cam[k] = p->cam[k];
    for (int k = 0; k < 3; ++k) { F.sky[k] = p->sky[k]; F.bg[k] = p->background[k]; }
    F.offset = p->normal_offset;
    F.seed = p->seed;
    F.width = p->width; F.height = p->height; F.jitter = p->jitter;
    F.integ = p->integrator; F.max_depth = p->max_depth;
    F.ao_count = p->ao_count; F.ao_length = p->ao_length;
    int64_t npix_total = (int64_t)p->width * p->height;
    F.pix_lo = p->pix_lo;
    int64_t hi = (p->pix_hi > 0) ? p->pix_hi : npix_total;
    F.npix = hi - p->pix_lo;
    F.tiled = (p->pix_lo % p->width == 0) && (hi % p->width == 0);
    F.row0 = p->pix_lo / p->width;
    F.row1 = hi / p->width;
    F.tiles_x = (p->width + 7) / 8;
    F.band_stride = p->band_stride > 0 ? p->band_stride : 1;
    F.band_offset = p->band_offset;
    if (!F.tiled) {
        F.band_stride = 1;
        F.band_offset = 0;
    }
    const int64_t trows = (F.row1 - F.row0 + 3) / 4;
    const int64_t mine = trows > F.band_offset ? (trows - F.band_offset + F.band_stride - 1) / F.band_stride : 0;
    F.nunits = F.tiled ? (int64_t)F.tiles_x * mine * 32 : F.npix;
    F.probe_budget = 0;
    F.epoch = 0;
    F.claims = nullptr;
    F.heavy_q = nullptr;
    F.probe_ctl = nullptr;
    F.probe_hint = nullptr;
    F.chunk = 0;
    F.nchunks = 1;
    F.chunk_done = nullptr;
    F.out64 = nullptr;
#if RT_TILE_PERM
    if (mine > 2) {
        // the integer nearest mine / phi that is coprime with mine (a bijection of the rows)
        auto gcd = [](int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a; };
        int64_t a = (int64_t)(0.6180339887498949 * (double)mine + 0.5);
        for (int64_t d = 0; d < mine; ++d) {
            if (a + d < mine && a + d > 0 && gcd(a + d, mine) == 1) { a = a + d; break; }
            if (a - d > 0 && gcd(a - d, mine) == 1) { a = a - d; break; }
        }
        F.perm_a = a;
    }
#endif
    if (F.tiled && F.band_stride > 1) {   // real pixels of this band set (ray counting)
        F.npix = 0;
        for (int64_t r = F.band_offset; r < trows; r += F.band_stride) {
            int64_t y0 = F.row0 + 4 * r, y1 = y0 + 4 < F.row1 ? y0 + 4 : F.row1;
            F.npix += (y1 - y0) * p->width;
        }
    }
    return F;
}

// walk-step budget of the eye frames' tile probe (0: no probe, row-major tiles): the
// RT_PROBE_BUDGET environment variable, else RT_PROBE_BUDGET; rt_set_probe_budget overrides
static std::atomic<int>& probe_budget_ref() {
    static std::atomic<int> b([] {
        const char* e = getenv("RT_PROBE_BUDGET");
        return e ? atoi(e) : RT_PROBE_BUDGET;
    }());
    return b;
}
static int probe_budget() { return probe_budget_ref().load(std::memory_order_relaxed); }

// device scratch for the wavefront, grown on demand and owned by the scene
struct WaveBuffers {
    int64_t cap = 0;
    void* mem = nullptr;
    int* d_sample = nullptr;
    unsigned long long* d_rays = nullptr;
    Wave W;
};

}  // namespace

// wavefront buffers per scene (keyed by scene pointer).  The map is shared by every
// context, so it has its own lock (a scene is destroyed without its context).
#include <map>
static std::map<rt_scene*, WaveBuffers>& wave_map() {
    static std::map<rt_scene*, WaveBuffers> m;
    return m;
}
static std::mutex& wave_lock() {
    static std::mutex m;
    return m;
}
void rt_render_release(rt_scene* s) {
    std::lock_guard<std::mutex> lk(wave_lock());
    auto& m = wave_map();
    auto it = m.find(s);
    if (it != m.end()) {
        cudaFree(it->second.mem);
        m.erase(it);
    }
}

static int ensure_wave(rt_scene* s, int64_t npix, WaveBuffers*& out) {
    std::lock_guard<std::mutex> lk(wave_lock());   // the entry stays put: std::map nodes are stable
    WaveBuffers& wb = wave_map()[s];
    if (wb.cap < npix) {
        if (wb.mem) cudaFree(wb.mem);
        size_t per = 32 + 16 + 16 + 16 + 16 + 8 + 4 + 4;
        size_t bytes = per * (size_t)npix + 64 * sizeof(unsigned) + 64;
        RT_CUDA_TRY(cudaMalloc(&wb.mem, bytes));
        char* p = (char*)wb.mem;
        wb.W.ray = (float4*)p; p += 32 * (size_t)npix;
        wb.W.thr = (float4*)p; p += 16 * (size_t)npix;
        wb.W.rad = (float4*)p; p += 16 * (size_t)npix;
        wb.W.rng = (uint2*)p; p += 16 * (size_t)npix;
        wb.W.hit = (float4*)p; p += 16 * (size_t)npix;
        wb.W.pix = (int64_t*)p; p += 8 * (size_t)npix;
        wb.W.queue[0] = (int*)p; p += 4 * (size_t)npix;
        wb.W.queue[1] = (int*)p; p += 4 * (size_t)npix;
        wb.W.count = (unsigned int*)p; p += 32 * sizeof(unsigned);
        wb.d_sample = (int*)p; p += 16;
        wb.d_rays = (unsigned long long*)p; p += 16;
        wb.cap = npix;
    }
    out = &wb;
    return RT_OK;
}

int rt_render_impl(rt_ctx* ctx, rt_scene* s, const rt_render_params* p, float* accum, uint64_t* rays_out,
                   double* out64) {
    FrameConst F = make_frame(p);
    const int64_t hi = (p->pix_hi > 0) ? p->pix_hi : (int64_t)p->width * p->height;
    if (F.pix_lo < 0 || hi <= F.pix_lo || hi > (int64_t)p->width * p->height) {
        rt_set_error("pixel range [%lld, %lld) outside the frame", (long long)p->pix_lo, (long long)hi);
        return RT_EINVAL;
    }
    if (p->band_stride < 0 || (p->band_stride > 0 && (p->band_offset < 0 || p->band_offset >= p->band_stride))) {
        rt_set_error("band_offset must be in [0, band_stride)");
        return RT_EINVAL;
    }
    if (p->s1 <= p->s0) {
        rt_set_error("empty sample window [%d, %d)", p->s0, p->s1);
        return RT_EINVAL;
    }
    if (F.nunits > 0x7FFFFFF0ll) {
        rt_set_error("too many work units (%lld) in one render", (long long)F.nunits);
        return RT_EINVAL;
    }
    if (F.nunits == 0 || F.npix == 0) {          // e.g. more GPUs than tile rows
        // the ray counter of this context reads 0 for this render (rt_multi_render sums it)
        RT_CUDA_TRY(cudaMemsetAsync(ctx->d_counter + 32, 0, sizeof(unsigned long long), ctx->stream));
        if (rays_out) *rays_out = 0;
        return RT_OK;
    }
    cudaStream_t st = ctx->stream;
    unsigned long long* d_rays = reinterpret_cast<unsigned long long*>(ctx->d_counter + 32);
    float4* acc = reinterpret_cast<float4*>(accum);
    if (p->kernel == RT_KERNEL_MEGA) {
        const int64_t ntiles = F.nunits >> 5;
        bool rb_replay = false;
        if (F.integ == RT_INTEG_EYE && F.tiled && probe_budget() > 0 && ntiles > 1) {
            if (ctx->probe_tiles < ntiles || ctx->probe_epoch == 0xFFFFFFFFu) {
                if (ctx->d_probe) RT_CUDA_TRY(cudaFree(ctx->d_probe));
                ctx->d_probe = nullptr;
                RT_CUDA_TRY(cudaMalloc(&ctx->d_probe, (size_t)ntiles * 12 + PC_WORDS * 4));
                RT_CUDA_TRY(cudaMemsetAsync(ctx->d_probe, 0, (size_t)ntiles * 12 + PC_WORDS * 4, st));
                ctx->probe_tiles = ntiles;
                ctx->probe_epoch = 0;
                ctx->lp_scene = nullptr;
            }
            F.probe_budget = probe_budget();
            F.epoch = ++ctx->probe_epoch;
            F.heavy_q = reinterpret_cast<unsigned long long*>(ctx->d_probe);
            F.claims = reinterpret_cast<unsigned*>(F.heavy_q + ctx->probe_tiles);
            F.probe_ctl = F.claims + ctx->probe_tiles;   // (zeroed by render_ctl_zero_kernel below)
            if (!s->probe_hint) {
                RT_CUDA_TRY(rt_alloc((void**)&s->probe_hint, sizeof(unsigned), st, false));
                RT_CUDA_TRY(cudaMemsetAsync(s->probe_hint, 0, sizeof(unsigned), st));
            }
            F.probe_hint = s->probe_hint;
            // the heavy-tile queue of this scene's last probe can be replayed when the tiles
            // are the same ones (scene, tile geometry and probe budget unchanged)
            const int64_t key[4] = {F.tiles_x * 1000003 + ntiles, F.row0 * 1000003 + F.row1,
                                    (int64_t)F.band_stride * 1000003 + F.band_offset, F.probe_budget};
            rb_replay = ctx->lp_scene == s && memcmp(ctx->lp_key, key, sizeof key) == 0;
            ctx->lp_scene = s;
            memcpy(ctx->lp_key, key, sizeof key);
        }
        if (F.integ != RT_INTEG_EYE && F.tiled && RT_PT_CHUNK > 0 && p->s1 - p->s0 > RT_PT_CHUNK && ntiles > 1) {
            if (ctx->chunk_tiles < ntiles) {
                if (ctx->d_chunk_done) RT_CUDA_TRY(cudaFree(ctx->d_chunk_done));
                ctx->d_chunk_done = nullptr;
                RT_CUDA_TRY(cudaMalloc(&ctx->d_chunk_done, sizeof(unsigned) * (size_t)ntiles));
                ctx->chunk_tiles = ntiles;
            }
            RT_CUDA_TRY(cudaMemsetAsync(ctx->d_chunk_done, 0, sizeof(unsigned) * (size_t)ntiles, st));
            F.chunk = RT_PT_CHUNK;
            F.nchunks = (p->s1 - p->s0 + RT_PT_CHUNK - 1) / RT_PT_CHUNK;
            F.chunk_done = reinterpret_cast<unsigned*>(ctx->d_chunk_done);
        }
        if (out64) {
            if (F.integ != RT_INTEG_EYE || F.nchunks > 1) {
                rt_set_error("float64 output is for eye frames");
                return RT_EINVAL;
            }
            F.out64 = reinterpret_cast<double4*>(out64);
        }
        // counters + probe words zeroed, then the frame: both launched with programmatic
        // stream serialization (each waits in-kernel for its predecessor: griddepcontrol.wait)
        cudaLaunchAttribute pdl[1];
        pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        pdl[0].val.programmaticStreamSerializationAllowed = RT_RENDER_PDL;
        {
            cudaLaunchConfig_t zc = {};
            zc.gridDim = dim3(1);
            zc.blockDim = dim3(256);
            zc.stream = st;
            zc.attrs = pdl;
            zc.numAttrs = 1;
            const unsigned ntiles_b = (unsigned)((ntiles + PROBE_BATCH - 1) / PROBE_BATCH * PROBE_BATCH);
            RT_CUDA_TRY(cudaLaunchKernelEx(&zc, render_ctl_zero_kernel, ctx->d_counter, F.probe_ctl, F.probe_hint,
                                           F.epoch, (int)(rb_replay && RT_PROBE_REPLAY), ntiles_b));
        }
        auto launch = [&](auto kern) -> int {
            int bps = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, MEGA_THREADS, 0);
            if (bps < 1) bps = 1;
            int64_t grid = (int64_t)ctx->num_sms * bps;
            int64_t want = (F.nunits + MEGA_THREADS - 1) / MEGA_THREADS;
            if (grid > want) grid = want;
            cudaLaunchConfig_t mc = {};
            mc.gridDim = dim3((unsigned)grid);
            mc.blockDim = dim3(MEGA_THREADS);
            mc.stream = st;
            mc.attrs = pdl;
            mc.numAttrs = 1;
            RT_CUDA_TRY(cudaLaunchKernelEx(&mc, kern, F, p->s0, p->s1, (const float4*)s->nodes, (const float4*)s->bvh4,
                                           (const float4*)s->tri_sorted, (const float4*)s->tri_attr,
                                           (const float4*)s->mat_color, (const float4*)s->mat_emissive,
                                           (const float4*)s->lights, s->n_lights, acc, ctx->d_counter, d_rays,
                                           ctx->d_error, rt_sphere_view(ctx, s, 0)));
            return RT_OK;
        };
        int rc;
        const bool sph = s->n_spheres > 0;   // triangle-only scenes run the walk without the sphere branch
        switch (F.integ) {
            case RT_INTEG_EYE:
                if (out64)
                    rc = sph ? launch(pt_megakernel<RT_INTEG_EYE, true, true>)
                             : launch(pt_megakernel<RT_INTEG_EYE, false, true>);
                else
                    rc = sph ? launch(pt_megakernel<RT_INTEG_EYE, true>) : launch(pt_megakernel<RT_INTEG_EYE, false>);
                break;
            case RT_INTEG_AO:
                rc = sph ? launch(pt_megakernel<RT_INTEG_AO, true>) : launch(pt_megakernel<RT_INTEG_AO, false>);
                break;
            case RT_INTEG_PTNEE:
                rc = sph ? launch(pt_megakernel<RT_INTEG_PTNEE, true>) : launch(pt_megakernel<RT_INTEG_PTNEE, false>);
                break;
            default:
                rc = sph ? launch(pt_megakernel<RT_INTEG_PT, true>) : launch(pt_megakernel<RT_INTEG_PT, false>);
                break;
        }
        if (rc) return rc;
    } else {
        if (out64) {
            rt_set_error("float64 output runs in the megakernel");
            return RT_EINVAL;
        }
        if (F.max_depth > 30) {
            rt_set_error("the wavefront kernel supports max_depth <= 30 (got %d); use kernel='mega'", F.max_depth);
            return RT_EINVAL;
        }
        RT_CUDA_TRY(cudaMemsetAsync(ctx->d_counter, 0, 64 * sizeof(unsigned int), st));
        WaveBuffers* wb;
        int rc = ensure_wave(s, F.nunits, wb);
        if (rc) return rc;
        RT_CUDA_TRY(cudaMemsetAsync(wb->d_sample, 0, 32, st));
        RT_CUDA_TRY(cudaMemcpyAsync(wb->d_sample, &p->s0, sizeof(int), cudaMemcpyHostToDevice, st));
        const bool sph = s->n_spheres > 0;
        int bps = 0;
        if (sph) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, wf_extend<true>, 128, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, wf_extend<false>, 128, 0);
        if (bps < 1) bps = 1;
        unsigned grid_ext = (unsigned)(ctx->num_sms * bps);
        unsigned grid_sh = (unsigned)ctx->num_sms * 8;
        int md = F.integ == RT_INTEG_EYE ? 1 : F.max_depth;
        // one wave (one sample index for every pixel) captured once as a CUDA graph
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        cudaStream_t cap;
        RT_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        RT_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        wf_raygen<<<grid_sh, WF_THREADS, 0, cap>>>(F, wb->d_sample, wb->W);
        for (int d = 0; d < md; ++d) {
            const SphereView sv = rt_sphere_view(ctx, s, 0);
            if (sph) {
                wf_extend<true><<<grid_ext, 128, 0, cap>>>(s->nodes, s->bvh4, s->tri_sorted, wb->W, d, ctx->d_counter,
                                                           ctx->d_error, sv);
                wf_shade<true><<<grid_sh, WF_THREADS, 0, cap>>>(F, s->tri_attr, s->mat_color, s->mat_emissive, wb->W,
                                                                d, sv);
            } else {
                wf_extend<false><<<grid_ext, 128, 0, cap>>>(s->nodes, s->bvh4, s->tri_sorted, wb->W, d,
                                                            ctx->d_counter, ctx->d_error, sv);
                wf_shade<false><<<grid_sh, WF_THREADS, 0, cap>>>(F, s->tri_attr, s->mat_color, s->mat_emissive,
                                                                 wb->W, d, sv);
            }
        }
        wf_accumulate<<<grid_sh, WF_THREADS, 0, cap>>>(F, wb->W, acc, wb->d_sample, ctx->d_counter, d_rays);
        cudaError_t ce = cudaStreamEndCapture(cap, &graph);
        if (ce != cudaSuccess) { cudaStreamDestroy(cap); RT_CUDA_TRY(ce); }
        ce = cudaGraphInstantiate(&exec, graph, 0);
        if (ce != cudaSuccess) { cudaGraphDestroy(graph); cudaStreamDestroy(cap); RT_CUDA_TRY(ce); }
        for (int smp = p->s0; smp < p->s1; ++smp) {
            ce = cudaGraphLaunch(exec, st);
            if (ce != cudaSuccess) break;
        }
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cap);
        RT_CUDA_TRY(ce);
        RT_CUDA_TRY(cudaGetLastError());
    }
    if (rays_out) {
        RT_CUDA_TRY(cudaMemcpyAsync(rays_out, d_rays, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        RT_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return RT_OK;
}

// render_frame in one call: the frame rendered from zero sums and delivered to the host as
// (npix, 4) float64 rows.  Eye frames in the megakernel write the float64 rows themselves;
// with n_chunks > 1 a whole eye frame renders in row chunks and each chunk's rows are copied
// out on the copy stream while the next chunk renders (the 32 B/pixel readback outlasts the
// render).  Every other frame renders into fp32 sums that are widened on the device and
// copied once.
int rt_render_host_impl(rt_ctx* ctx, rt_scene* s, const rt_render_params* p, double* host_out, int n_chunks,
                        uint64_t* rays_out) {
    const int64_t npix = (int64_t)p->width * p->height;
    const int stride = p->band_stride > 1 ? p->band_stride : 1;
    const bool whole = p->pix_lo == 0 && (p->pix_hi == 0 || p->pix_hi == npix);
    const bool direct = p->integrator == RT_INTEG_EYE && p->kernel == RT_KERNEL_MEGA;
    int nc = direct && whole && !rays_out && n_chunks > 1 ? n_chunks : 1;
    if (nc > 8) nc = 8;
    if ((int64_t)p->height < 8LL * stride * nc) nc = 1;
    cudaStream_t st = ctx->stream;
    if (ctx->rb_pix < npix) {           // float64 rows + fp32 sums, grown on demand
        if (ctx->d_rb) RT_CUDA_TRY(cudaFree(ctx->d_rb));
        ctx->d_rb = nullptr;
        ctx->rb_pix = 0;
        RT_CUDA_TRY(cudaMalloc(&ctx->d_rb, 48 * (size_t)npix));
        ctx->rb_pix = npix;
    }
    double* out64 = reinterpret_cast<double*>(ctx->d_rb);
    float* acc32 = reinterpret_cast<float*>(out64 + 4 * ctx->rb_pix);
    unsigned long long* d_rays = reinterpret_cast<unsigned long long*>(ctx->d_counter + 32);
    if (direct) {
        // pixels outside the band set / pixel range stay 0 (the kernel writes only its own)
        if (!whole || stride > 1) RT_CUDA_TRY(cudaMemsetAsync(out64, 0, 32 * (size_t)npix, st));
        if (nc == 1) {
            int rc = rt_render_impl(ctx, s, p, nullptr, nullptr, out64);
            if (rc) return rc;
            RT_CUDA_TRY(cudaMemcpyAsync(host_out, out64, 32 * (size_t)npix, cudaMemcpyDeviceToHost, st));
        } else {
            int rc = rt_io_streams(ctx);
            if (rc) return rc;
            cudaStream_t cp = ctx->io_out;
            // chunks of whole 4-row tile bands (multiples of 4 * stride rows keep every band)
            const int64_t rows = ((int64_t)p->height + 4LL * stride * nc - 1) / (4LL * stride * nc) * 4 * stride;
            int k = 0;
            for (int64_t r0 = 0; r0 < p->height; r0 += rows, ++k) {
                const int64_t r1 = r0 + rows < p->height ? r0 + rows : p->height;
                rt_render_params q = *p;
                q.pix_lo = r0 * p->width;
                q.pix_hi = r1 * p->width;
                rc = rt_render_impl(ctx, s, &q, nullptr, nullptr, out64);
                if (rc) return rc;
                RT_CUDA_TRY(cudaEventRecord(ctx->io_ev[k], st));
                RT_CUDA_TRY(cudaStreamWaitEvent(cp, ctx->io_ev[k], 0));
                RT_CUDA_TRY(cudaMemcpyAsync(host_out + 4 * q.pix_lo, out64 + 4 * q.pix_lo,
                                            32 * (size_t)(q.pix_hi - q.pix_lo), cudaMemcpyDeviceToHost, cp));
            }
            RT_CUDA_TRY(cudaEventRecord(ctx->io_ev[8], cp));
            RT_CUDA_TRY(cudaStreamWaitEvent(st, ctx->io_ev[8], 0));   // later work follows the copies
        }
    } else {
        RT_CUDA_TRY(cudaMemsetAsync(acc32, 0, 16 * (size_t)npix, st));
        int rc = rt_render_impl(ctx, s, p, acc32, nullptr);
        if (rc) return rc;
        widen_kernel<<<ctx->num_sms * 8, 256, 0, st>>>(reinterpret_cast<const float4*>(acc32),
                                                        reinterpret_cast<double4*>(out64), npix);
        RT_CUDA_TRY(cudaGetLastError());
        RT_CUDA_TRY(cudaMemcpyAsync(host_out, out64, 32 * (size_t)npix, cudaMemcpyDeviceToHost, st));
    }
    if (rays_out) RT_CUDA_TRY(cudaMemcpyAsync(rays_out, d_rays, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    int err = 0;                                // the device error flag rides on the same sync
    RT_CUDA_TRY(cudaMemcpyAsync(&err, ctx->d_error, sizeof err, cudaMemcpyDeviceToHost, st));
    RT_CUDA_TRY(cudaStreamSynchronize(st));
    return err ? rt_check_device_error(ctx) : RT_OK;
}

int rt_resolve_impl(rt_ctx* ctx, const float* accum, int64_t npix, int gamma, uint8_t* rgb) {
    resolve_kernel<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(reinterpret_cast<const float4*>(accum), npix, gamma,
                                                             rgb, ctx->d_error);
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

int rt_raygen_impl(rt_ctx* ctx, const rt_render_params* p, int sample, float* rays) {
    FrameConst F = make_frame(p);
    raygen_kernel<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(F, sample, reinterpret_cast<float4*>(rays));
    RT_CUDA_TRY(cudaGetLastError());
    return RT_OK;
}

// ---- RNG stream known-answer hook (tests): the first n raw PCG32 outputs of the
// (seed, pixel, sample) stream the kernels draw from (sampling.py:38-79, 124-127) ----
namespace {
__global__ void stream_draws_kernel(uint64_t seed, uint64_t pix, uint64_t s, int n, uint32_t* out) {
    uint64_t state, inc;
    rt_stream_for(seed, pix, s, state, inc);
    for (int k = 0; k < n; ++k) out[k] = rt_pcg_next(state, inc);
}
}  // namespace

extern "C" int rt_stream_draws(rt_ctx* c, uint64_t seed, uint64_t pixel, uint64_t sample, int32_t n,
                               uint32_t* out) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(out && n >= 0 && n <= 4096, "bad output buffer");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    uint32_t* d = nullptr;
    RT_CUDA_TRY(rt_alloc((void**)&d, sizeof(uint32_t) * (n > 0 ? n : 1), c->stream, false));
    stream_draws_kernel<<<1, 1, 0, c->stream>>>(seed, pixel, sample, n, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, c->stream);
    rt_free(d, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        rt_set_error("rt_stream_draws: %s", cudaGetErrorString(e));
        return RT_ECUDA;
    }
    return RT_OK;
}

#if RT_TIMELINE
extern "C" int rt_debug_timeline(unsigned long long* out, int32_t n_warps) {
    RT_CHECK_ARG(out && n_warps > 0 && n_warps <= RT_TIMELINE_WARPS, "bad timeline buffer");
    RT_CUDA_TRY(cudaDeviceSynchronize());
    RT_CUDA_TRY(cudaMemcpyFromSymbol(out, g_timeline, sizeof(unsigned long long) * 4 * n_warps));
    return RT_OK;
}
#endif

extern "C" int rt_set_probe_budget(int32_t budget, int32_t* previous) {
    RT_CHECK_ARG(budget >= 0, "the probe budget is a walk-step count >= 0 (0: no probe)");
    const int old = probe_budget_ref().exchange(budget);
    if (previous) *previous = old;
    return RT_OK;
}

extern "C" int rt_probe_stats(rt_ctx* c, uint32_t* out4) {
    RT_CTX_LOCK(c);
    RT_CHECK_ARG(out4, "NULL output");
    RT_CUDA_TRY(cudaSetDevice(c->device));
    for (int k = 0; k < 4; ++k) out4[k] = 0;
    if (!c->d_probe) return RT_OK;
    const unsigned* pc = reinterpret_cast<const unsigned*>(reinterpret_cast<const char*>(c->d_probe) +
                                                           (size_t)c->probe_tiles * 12);
    const int idx[4] = {PC_DONE, PC_TAIL, PC_HEAD, PC_LIMIT};
    for (int k = 0; k < 4; ++k)
        RT_CUDA_TRY(cudaMemcpyAsync(out4 + k, pc + idx[k], 4, cudaMemcpyDeviceToHost, c->stream));
    RT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return RT_OK;
}
