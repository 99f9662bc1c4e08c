// On-device world construction, sm_100a.
//
// The reference builds every world of a batch with O(W) Python loops at
// engine construction: build_world_batch (world.py:82-194: segmentize,
// scene_segments, grid_offsets, assign_scenes, the padded (W, P_max) arrays),
// the spawn table (engine.py:192-227 over filter_agents, scenario.py:169-192),
// _compact_subset (engine.py:234-253) and eval.random_goals' arc-length goal
// resampling (config.py:222-278).  Here they are three launches:
//
//   dg_build_scenes  one CTA per scene: point pairs -> kept segments with a
//                    block-wide ordered compaction (ballot + warp-total scan),
//                    the lane / road-edge subsets as scene-local index lists,
//                    the cumulative arc length at every polyline vertex, and the
//                    spawn filter over the scene's agent records (one warp,
//                    ballots in file order, first `cap`).
//   dg_build_worlds  one thread per (world, agent) slot: scene assignment,
//                    grid offset, spawn table and initial state straight into
//                    the engine's device arrays; optional per-(world, segment)
//                    padded WorldBatch arrays and per-(world, k) lane / edge
//                    subsets in global coordinates.
//                    With random goals: one thread per valid slot walks its
//                    nearest lane polyline by arc length.
//
// Arithmetic is the reference's term for term (-fmad=false; IEEE sqrt and
// division), so every output is bit-identical to the host build, which is
// itself pinned to the reference (tests/golden/init_default.npz,
// goals_random.npz, worlds_4096.npz).  math.dist in the spawn filter is
// CPython's vector_norm (Modules/mathmodule.c), restated below.

#include <cstdint>
#include <cstdio>
#include <cmath>

#include <cuda_runtime.h>

#include "drivegrid_b200.h"

int dg_internal_fail(int code, const char* msg);
int dg_internal_cuda_fail(cudaError_t e, const char* where);

namespace {

constexpr int kSceneThreads = 256;
constexpr int kSceneWarps = kSceneThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ bool is_lane(int code) { return code == 1 || code == 2; }      // LANE_CENTER_CODES
__device__ __forceinline__ bool is_edge(int code) { return code == 15 || code == 16; }    // ROAD_EDGE_CODES

// pairs (= candidate segments) before scene s: every polyline of n points has n - 1
__device__ __forceinline__ int pair_base(const DgScenePool& P, int s) {
    return P.poly_start[P.scene_poly[s]] - P.scene_poly[s];
}

// ---- CPython 3.12 math.dist(p, q) for 2-D points: vector_norm over |p - q|
//      with the scaled double-length accumulation and the differential
//      correction (mathmodule.c), exact products by fma.
struct DL { double hi, lo; };
__device__ __forceinline__ DL dl_mul(double x, double y) {
    const double z = x * y;
    return {z, __fma_rn(x, y, -z)};
}
__device__ __forceinline__ DL dl_fast_sum(double a, double b) {
    const double hi = a + b;
    return {hi, (a - hi) + b};
}
__device__ double py_dist2(double px, double py, double qx, double qy) {
    double v[2] = {fabs(px - qx), fabs(py - qy)};
    double mx = 0.0;
    bool nan = false;
    for (int i = 0; i < 2; ++i) {
        nan |= v[i] != v[i];
        if (v[i] > mx) mx = v[i];
    }
    if (isinf(mx)) return mx;
    if (nan) return NAN;
    if (mx == 0.0) return mx;
    double outer = 1.0;
    int e;
    frexp(mx, &e);
    if (e < -1023) {   // subnormal maximum: rescale once (DBL_MIN), as the recursion does
        const double dmin = 2.2250738585072014e-308;
        v[0] /= dmin;
        v[1] /= dmin;
        mx /= dmin;
        outer = dmin;
        frexp(mx, &e);
    }
    const double scale = ldexp(1.0, -e);
    double csum = 1.0, f1 = 0.0, f2 = 0.0;
    for (int i = 0; i < 2; ++i) {
        const double x = v[i] * scale;
        const DL pr = dl_mul(x, x);
        const DL sm = dl_fast_sum(csum, pr.hi);
        csum = sm.hi;
        f1 += pr.lo;
        f2 += sm.lo;
    }
    double h = sqrt(csum - 1.0 + (f1 + f2));
    const DL pr = dl_mul(-h, h);
    const DL sm = dl_fast_sum(csum, pr.hi);
    csum = sm.hi;
    f1 += pr.lo;
    f2 += sm.lo;
    const double x = csum - 1.0 + (f1 + f2);
    h += x / (2.0 * h);
    return outer * (h / scale);
}

// Python's max(a, b, c, d): keeps the earlier value unless a later one compares greater
__device__ __forceinline__ double py_max4(double a, double b, double c, double d) {
    double m = a;
    if (b > m) m = b;
    if (c > m) m = c;
    if (d > m) m = d;
    return m;
}

// exclusive block scan of three 0/1 flags (kSceneThreads threads); returns the
// block totals through `tot`
__device__ __forceinline__ void block_scan3(int f0, int f1, int f2, int* ex, int* tot, int (*sw)[3]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned b[3] = {__ballot_sync(kFull, f0), __ballot_sync(kFull, f1), __ballot_sync(kFull, f2)};
    if (lane == 0)
        for (int i = 0; i < 3; ++i) sw[warp][i] = __popc(b[i]);
    __syncthreads();
    for (int i = 0; i < 3; ++i) {
        int before = 0, all = 0;
        for (int k = 0; k < kSceneWarps; ++k) {
            before += k < warp ? sw[k][i] : 0;
            all += sw[k][i];
        }
        ex[i] = before + __popc(b[i] & lt);
        tot[i] = all;
    }
    __syncthreads();
}

// ---- dg_build_scenes: one CTA per scene
__global__ void __launch_bounds__(kSceneThreads) scene_build_kernel(const DgScenePool P, const DgSceneBuild B,
                                                                   DgSceneSegments O) {
    __shared__ int sw[kSceneWarps][3];
    const int s = blockIdx.x;
    const int tid = threadIdx.x;
    const int j0 = P.scene_poly[s], j1 = P.scene_poly[s + 1];
    const int p0 = P.poly_start[j0], p1 = P.poly_start[j1];
    const int base = p0 - j0;
    const double bh = B.bbox_half;

    // (1) segmentize (world.py:82-109) + scene_segments' polyline order (111-121):
    //     pair (p, p + 1) of a polyline, kept if 0 < |b - a| <= gap and both
    //     endpoints inside the box; ordered compaction over the scene's points
    int run[3] = {0, 0, 0};
    for (int c0 = p0; c0 < p1; c0 += kSceneThreads) {
        const int p = c0 + tid;
        int keep = 0, code = 0;
        double ax = 0.0, ay = 0.0, dx = 0.0, dy = 0.0, dist = 0.0;
        if (p < p1) {
            int lo = j0, hi = j1 - 1;            // polyline of p: last j with poly_start[j] <= p
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (P.poly_start[mid] <= p) lo = mid; else hi = mid - 1;
            }
            if (p + 1 < P.poly_start[lo + 1]) {
                code = P.poly_type[lo];
                ax = P.points[2 * p];
                ay = P.points[2 * p + 1];
                const double bx = P.points[2 * p + 2], by = P.points[2 * p + 3];
                dx = bx - ax;
                dy = by - ay;
                dist = sqrt(dx * dx + dy * dy);
                const bool inside = (fabs(ax) <= bh && fabs(ay) <= bh) && (fabs(bx) <= bh && fabs(by) <= bh);
                keep = (dist > 0.0) && (dist <= B.gap) && inside;
                if (keep) {
                    // midpoint 0.5 * (a + b), direction diff / dist, half length 0.5 * dist
                    ax = 0.5 * (ax + bx);
                    ay = 0.5 * (ay + by);
                }
            }
        }
        const int lane_f = keep && is_lane(code), edge_f = keep && is_edge(code);
        int ex[3], tot[3];
        block_scan3(keep, lane_f, edge_f, ex, tot, sw);
        if (keep) {
            const int q = run[0] + ex[0];        // scene-local segment index
            const int64_t r = int64_t(base) + q;
            O.mid[2 * r] = ax;
            O.mid[2 * r + 1] = ay;
            O.dir[2 * r] = dx / dist;
            O.dir[2 * r + 1] = dy / dist;
            O.type[r] = code;
            O.half_len[r] = 0.5 * dist;
            O.half_wid[r] = B.half_width;
            if (lane_f) O.lane_index[base + run[1] + ex[1]] = q;
            if (edge_f) O.edge_index[base + run[2] + ex[2]] = q;
        }
        for (int i = 0; i < 3; ++i) run[i] += tot[i];
    }

    // (2) cumulative arc length at every vertex of every polyline (config.py:222-236,
    //     np.cumsum: one sequential sum per polyline) and the scene's lane count
    int lanes = 0;
    for (int j = j0 + tid; j < j1; j += kSceneThreads) {
        const int a = P.poly_start[j], b = P.poly_start[j + 1];
        double acc = 0.0;
        if (a < b) O.arc[a] = 0.0;
        for (int p = a; p + 1 < b; ++p) {
            const double sx = P.points[2 * p + 2] - P.points[2 * p];
            const double sy = P.points[2 * p + 3] - P.points[2 * p + 1];
            acc = acc + sqrt(sx * sx + sy * sy);
            O.arc[p + 1] = acc;
        }
        lanes += is_lane(P.poly_type[j]);
    }
    for (int o = 16; o > 0; o >>= 1) lanes += __shfl_xor_sync(kFull, lanes, o);
    if ((tid & 31) == 0) sw[tid >> 5][0] = lanes;
    __syncthreads();

    // (3) filter_agents (scenario.py:169-192): in-box endpoints, start-goal
    //     distance above goal_radius, file order, first `cap`
    if (tid < 32) {
        const int a0 = P.scene_agent[s], a1 = P.scene_agent[s + 1];
        int kept = 0;
        for (int c0 = a0; c0 < a1 && kept < B.cap; c0 += 32) {
            const int a = c0 + tid;
            bool ok = false;
            if (a < a1) {
                const double* r = P.agents + 7 * int64_t(a);
                const double sx = r[0], sy = r[1], gx = r[3], gy = r[4];
                ok = !(py_max4(fabs(sx), fabs(sy), fabs(gx), fabs(gy)) > bh) &&
                     !(py_dist2(sx, sy, gx, gy) <= B.goal_radius);
            }
            const unsigned bal = __ballot_sync(kFull, ok);
            const int slot = kept + __popc(bal & ((1u << tid) - 1u));
            if (ok && slot < B.cap) O.kept_agent[P.scene_agent[s] + slot] = a;
            kept += __popc(bal);
        }
        if (tid == 0) {
            int nl = 0;
            for (int k = 0; k < kSceneWarps; ++k) nl += sw[k][0];
            O.seg_count[s] = run[0];
            O.lane_count[s] = run[1];
            O.edge_count[s] = run[2];
            O.kept_count[s] = kept < B.cap ? kept : B.cap;
            O.lane_polys[s] = nl;
        }
    }
}

// ---- dg_build_worlds: one thread per (world, agent slot)
__device__ __forceinline__ void world_origin(const DgWorldBuild& B, int w, int* scene, double* ox, double* oy) {
    const int64_t g = B.world_base + w;
    *scene = B.scene_order[g % B.num_scenes];
    *ox = double(g % B.grid_cols) * B.pitch;      // grid_offsets (world.py:124-128)
    *oy = double(g / B.grid_cols) * B.pitch;
}

__global__ void spawn_kernel(const DgScenePool P, const DgSceneSegments S, const DgWorldBuild B) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t WM = int64_t(B.W) * B.M;
    if (i >= WM) return;
    const int w = int(i / B.M), m = int(i % B.M);
    int s;
    double ox, oy;
    world_origin(B, w, &s, &ox, &oy);
    if (m == 0) {
        B.assignment[w] = s;
        B.grid_offset[2 * w] = ox;
        B.grid_offset[2 * w + 1] = oy;
    }
    if (!B.valid) return;   // world arrays only
    // spawn table (engine.py:192-227): the scene's kept agents, then parked slots
    double st[DG_NUM_STATE];
#pragma unroll
    for (int f = 0; f < DG_NUM_STATE; ++f) st[f] = 0.0;
    st[10] = 1.0;   // brake_sign_front
    st[11] = 1.0;   // brake_sign_rear
    double len = 4.0, wid = 2.0, sxg = 0.0, syg = 0.0, gxg = 0.0, gyg = 0.0, yaw = 0.0;
    const bool valid = m < S.kept_count[s];
    if (valid) {
        const double* r = P.agents + 7 * int64_t(S.kept_agent[P.scene_agent[s] + m]);
        sxg = r[0] + ox;
        syg = r[1] + oy;
        gxg = r[3] + ox;
        gyg = r[4] + oy;
        yaw = r[2];
        len = r[5];
        wid = r[6];
        st[0] = sxg;
        st[1] = syg;
        st[2] = yaw;
    } else {
        st[0] = ox + B.offstage_x;
        st[1] = oy;
    }
#pragma unroll
    for (int f = 0; f < DG_NUM_STATE; ++f) B.state[int64_t(f) * WM + i] = st[f];
    B.valid[i] = valid;
    if (B.alive) B.alive[i] = valid;
    B.start_xy[2 * i] = sxg;
    B.start_xy[2 * i + 1] = syg;
    B.goal_xy[2 * i] = gxg;
    B.goal_xy[2 * i + 1] = gyg;
    B.start_yaw[i] = yaw;
    B.length[i] = len;
    B.width[i] = wid;
    // circle_layout (observation.py:44-48)
    const double wr = 0.55 * wid;
    const double r = 0.45 > wr ? 0.45 : wr;
    const double t = len / 2.0 - 0.8 * r;
    const double d0 = 0.0 > t ? 0.0 : t;
    const double half_wb = B.wheelbase / 2.0;
    B.r_hull[i] = r;
    B.d_hull[i] = half_wb < d0 ? half_wb : d0;
}

// padded WorldBatch (world.py:148-194): one thread per (world, segment slot)
__global__ void padded_kernel(const DgScenePool P, const DgSceneSegments S, const DgWorldBuild B) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n = int64_t(B.W) * B.p_max;
    if (i >= n) return;
    const int w = int(i / B.p_max), p = int(i % B.p_max);
    const int s = B.scene_order[(B.world_base + w) % B.num_scenes];
    const bool in = p < S.seg_count[s];
    const int64_t r = int64_t(pair_base(P, s)) + p;
    B.wb_mid[2 * i] = in ? S.mid[2 * r] : 0.0;
    B.wb_mid[2 * i + 1] = in ? S.mid[2 * r + 1] : 0.0;
    B.wb_dir[2 * i] = in ? S.dir[2 * r] : 0.0;
    B.wb_dir[2 * i + 1] = in ? S.dir[2 * r + 1] : 0.0;
    B.wb_type[i] = in ? S.type[r] : 0;
    B.wb_half_len[i] = in ? S.half_len[r] : 0.0;
    B.wb_half_wid[i] = in ? S.half_wid[r] : 0.0;
    B.wb_mask[i] = in;
}

// _compact_subset (engine.py:234-253): lane (sub = 0) or edge (sub = 1) segments
// of each world, dense [W][K], midpoints in global coordinates
__global__ void subset_kernel(const DgScenePool P, const DgSceneSegments S, const DgWorldBuild B, int sub) {
    const int K = sub ? B.k_edge : B.k_lane;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= int64_t(B.W) * K) return;
    const int w = int(i / K), k = int(i % K);
    int s;
    double ox, oy;
    world_origin(B, w, &s, &ox, &oy);
    const int base = pair_base(P, s);
    const bool in = k < (sub ? S.edge_count[s] : S.lane_count[s]);
    const int64_t r = in ? int64_t(base) + (sub ? S.edge_index : S.lane_index)[base + k] : 0;
    double* mid = sub ? B.edge_mid : B.lane_mid;
    double* dir = sub ? B.edge_dir : B.lane_dir;
    mid[2 * i] = in ? S.mid[2 * r] + ox : 0.0;
    mid[2 * i + 1] = in ? S.mid[2 * r + 1] + oy : 0.0;
    dir[2 * i] = in ? S.dir[2 * r] : 0.0;
    dir[2 * i + 1] = in ? S.dir[2 * r + 1] : 0.0;
    (sub ? B.edge_half_len : B.lane_half_len)[i] = in ? S.half_len[r] : 0.0;
    (sub ? B.edge_half_wid : B.lane_half_wid)[i] = in ? S.half_wid[r] : 0.0;
    (sub ? B.edge_mask : B.lane_mask)[i] = in;
}

// eval.random_goals (config.py:222-278): one thread per (world, agent) slot.  The
// distance draws come from the host's Philox stream (seed, 4) in (world, agent)
// order, one per valid agent of a scene with lanes: draw index = q * C +
// prefix[r] + m for global world g = q * S + r (C = draws per full cycle of the
// scene order, prefix[r] = draws of its first r worlds).
__global__ void goals_kernel(const DgScenePool P, const DgSceneSegments S, const DgWorldBuild B) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= int64_t(B.W) * B.M) return;
    const int w = int(i / B.M), m = int(i % B.M);
    int s;
    double ox, oy;
    world_origin(B, w, &s, &ox, &oy);
    if (m >= S.kept_count[s] || S.lane_polys[s] == 0) return;
    double reach = B.goal_min;
    if (B.goal_min != B.goal_max) {
        const int64_t g = B.world_base + w;
        const int64_t q = g / B.num_scenes, rr = g % B.num_scenes;
        int64_t cyc = 0, pre = 0;
        for (int j = 0; j < B.num_scenes; ++j) {
            const int sj = B.scene_order[j];
            const int c = S.lane_polys[sj] ? S.kept_count[sj] : 0;
            cyc += c;
            pre += j < rr ? c : 0;
        }
        reach = B.goal_draws[q * cyc + pre + m];
    }
    // scene-local start exactly as the reference forms it: start_xy - offset
    const double lx = B.start_xy[2 * i] - ox, ly = B.start_xy[2 * i + 1] - oy;
    // nearest vertex over the lane polylines (argmin per lane, earlier lane on ties)
    double best = 0.0;
    int pick = -1, vert = 0;
    for (int j = P.scene_poly[s]; j < P.scene_poly[s + 1]; ++j) {
        if (!is_lane(P.poly_type[j])) continue;
        const int a = P.poly_start[j], b = P.poly_start[j + 1];
        double vmin = 0.0;
        int v = -1;
        for (int p = a; p < b; ++p) {
            const double dx = P.points[2 * p] - lx, dy = P.points[2 * p + 1] - ly;
            const double d2 = dx * dx + dy * dy;
            if (v < 0 || d2 < vmin || (d2 != d2 && vmin == vmin)) { vmin = d2; v = p; }
        }
        if (pick < 0 || vmin < best) { best = vmin; pick = j; vert = v; }
    }
    if (pick < 0 || vert < 0) return;
    const int a = P.poly_start[pick], b = P.poly_start[pick + 1];
    const double arc0 = S.arc[vert];
    const double arc_end = S.arc[b - 1];
    // polyline_arc_point: forward, then backward
    for (int dirn = 0; dirn < 2; ++dirn) {
        const double target = arc0 + (dirn ? -reach : reach);
        if (!(target >= 0.0 && target <= arc_end)) continue;
        int cnt = 0;                                  // searchsorted(arc, target, 'right')
        for (int p = a; p < b; ++p) cnt += S.arc[p] <= target;
        int k = cnt - 1;
        if (k > b - a - 2) k = b - a - 2;
        const int p = a + k;
        const double sx = P.points[2 * p + 2] - P.points[2 * p];
        const double sy = P.points[2 * p + 3] - P.points[2 * p + 1];
        const double len = sqrt(sx * sx + sy * sy);
        const double along = len > 0.0 ? (target - S.arc[p]) / len : 0.0;
        const double gx = P.points[2 * p] + along * sx, gy = P.points[2 * p + 1] + along * sy;
        B.goal_xy[2 * i] = gx + ox;
        B.goal_xy[2 * i + 1] = gy + oy;
        return;
    }
}

int launch_status(const char* where) {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DG_OK : dg_internal_cuda_fail(e, where);
}

}  // namespace

extern "C" {

int dg_build_scenes(const DgScenePool* pool, const DgSceneBuild* build, DgSceneSegments* out, void* stream) {
    if (!pool || !build || !out) return dg_internal_fail(DG_EINVAL, "dg_build_scenes: null argument");
    if (pool->num_scenes < 1) return dg_internal_fail(DG_EINVAL, "dg_build_scenes: empty scene list");
    if (build->cap < 0) return dg_internal_fail(DG_EINVAL, "dg_build_scenes: cap < 0");
    if (!pool->points || !pool->poly_start || !pool->poly_type || !pool->scene_poly || !pool->scene_agent ||
        (pool->num_agents > 0 && !pool->agents))
        return dg_internal_fail(DG_EINVAL, "dg_build_scenes: missing pool array");
    if (!out->mid || !out->dir || !out->type || !out->half_len || !out->half_wid || !out->lane_index ||
        !out->edge_index || !out->arc || !out->seg_count || !out->lane_count || !out->edge_count ||
        !out->kept_count || !out->kept_agent || !out->lane_polys)
        return dg_internal_fail(DG_EINVAL, "dg_build_scenes: missing output array");
    scene_build_kernel<<<pool->num_scenes, kSceneThreads, 0, static_cast<cudaStream_t>(stream)>>>(*pool, *build,
                                                                                                 *out);
    return launch_status("dg_build_scenes");
}

int dg_build_worlds(const DgScenePool* pool, const DgSceneSegments* scenes, const DgWorldBuild* b, void* stream) {
    if (!pool || !scenes || !b) return dg_internal_fail(DG_EINVAL, "dg_build_worlds: null argument");
    if (b->W < 1 || b->M < 1 || b->num_scenes != pool->num_scenes || b->grid_cols < 1 || b->world_base < 0)
        return dg_internal_fail(DG_EINVAL, "dg_build_worlds: bad dimensions");
    if (!b->scene_order || !b->assignment || !b->grid_offset)
        return dg_internal_fail(DG_EINVAL, "dg_build_worlds: missing scene_order / assignment / grid_offset");
    if (b->valid && (!b->start_xy || !b->goal_xy || !b->start_yaw || !b->length || !b->width || !b->r_hull ||
                     !b->d_hull || !b->state))
        return dg_internal_fail(DG_EINVAL, "dg_build_worlds: the spawn table needs every spawn array");
    if (b->random_goals && (!b->start_xy || !b->goal_xy))
        return dg_internal_fail(DG_EINVAL, "dg_build_worlds: random goals need start_xy and goal_xy");
    if (b->random_goals && b->goal_min != b->goal_max && !b->goal_draws)
        return dg_internal_fail(DG_EINVAL, "dg_build_worlds: random goals need goal_draws");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t WM = int64_t(b->W) * b->M;
    spawn_kernel<<<unsigned((WM + 255) / 256), 256, 0, st>>>(*pool, *scenes, *b);
    if (int rc = launch_status("dg_build_worlds(spawn)")) return rc;
    if (b->random_goals) {
        goals_kernel<<<unsigned((WM + 127) / 128), 128, 0, st>>>(*pool, *scenes, *b);
        if (int rc = launch_status("dg_build_worlds(goals)")) return rc;
    }
    if (b->p_max > 0) {
        if (!b->wb_mid || !b->wb_dir || !b->wb_type || !b->wb_half_len || !b->wb_half_wid || !b->wb_mask)
            return dg_internal_fail(DG_EINVAL, "dg_build_worlds: p_max > 0 needs every wb_* array");
        const int64_t n = int64_t(b->W) * b->p_max;
        padded_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(*pool, *scenes, *b);
        if (int rc = launch_status("dg_build_worlds(padded)")) return rc;
    }
    for (int sub = 0; sub < 2; ++sub) {
        const int K = sub ? b->k_edge : b->k_lane;
        if (K <= 0) continue;
        const bool ok = sub ? (b->edge_mid && b->edge_dir && b->edge_half_len && b->edge_half_wid && b->edge_mask)
                            : (b->lane_mid && b->lane_dir && b->lane_half_len && b->lane_half_wid && b->lane_mask);
        if (!ok) return dg_internal_fail(DG_EINVAL, "dg_build_worlds: k_lane / k_edge > 0 needs the subset arrays");
        const int64_t n = int64_t(b->W) * K;
        subset_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(*pool, *scenes, *b, sub);
        if (int rc = launch_status("dg_build_worlds(subset)")) return rc;
    }
    return DG_OK;
}

}  // extern "C"
