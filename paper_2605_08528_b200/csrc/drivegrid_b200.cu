// drivegrid_b200.cu -- the batched multi-world, multi-agent vehicle step on
// B200 (sm_100a): one fused kernel per 30 Hz control tick.
//
// Mapping: one CTA per world, one warp per agent slot (M <= 16 warps).
//   phase 0  action finiteness scan for the world (block vote)           engine.py:286-295
//   phase 1  warp 0, lane m: agent m state -> registers, decode, 4x
//            single-track substeps (or 1 bicycle step), alive mask       engine.py:410-421,
//                                                                        vehicle.py:162-336
//            meanwhile: TMA bulk copy of the world's scene geometry
//            (cp.async.bulk, mbarrier complete_tx) into shared memory
//   phase 2  warp m: road k-select by ballot compaction, neighbours with
//            stable rank + swept 3x3-circle TTC, ego block            observation.py:51-293
//            nearest lane (warp argmin), edge TTC, edge OBB test,
//            hull contact (warp vote), dense terms, events, priority  rewards.py:78-268,
//                                                                        engine.py:472-509
//            tail: timeout, park, alive (+ optional fused autoreset)  engine.py:370-406
//            the agent's 1929-float observation row, streamed with
//            16-byte st.global.cs from a lane-parallel generator
//
// Numerics: float64 throughout in the reference's global coordinates, and
// the translation unit is compiled with -fmad=false: every a*b+c rounds twice
// exactly as numpy evaluates it, so sqrt/div/mul/add results and therefore
// every threshold decision (d2 <= r^2, d2 < (ra+rb)^2, dist <= 3, ...) are
// bit-identical to the reference.  Only libm transcendentals (sin, cos,
// atan2, exp, tan) may differ from the host's in the last ulp.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <unistd.h>
#include <new>

#include "dg_fastmath.cuh"
#include "drivegrid_b200.h"

namespace {

constexpr int kMaxAgents = 16;
constexpr int kZeroChunk = 4096;   // bytes of zeros in shared memory, source of the TMA row clears
constexpr int kPfxSlots = 16;      // resident rings up to this many slots keep the world's prefix record in smem
constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kBitFinished = 32u;   // finalize_agent: done or timed out this tick

enum StateField {
    SX = 0, SY, SYAW, SVX, SVY, SOM, SANG, SRATE, SWF, SWR, SBF, SBR
};

// Refined reciprocals (dg::drcp_refined) of the constant divisors, computed once
// on the device at engine creation: a division by a constant becomes
// dg::ddiv_y(a, b, rc.b) -- the same value ddiv(a, b) computes, without the
// reciprocal's five dependent FMAs on every use (kernel-parameter constants).
struct Rcp {
    double steer_inertia, wheel_radius, chassis_mass, yaw_inertia, i_axle, wheelbase;
    double bbox_half, speed_norm, pi, ttc_max, road_radius, lane_sigma;
};

__device__ __forceinline__ Rcp make_rcp(const DgConsts& k) {
    Rcp r;
    r.steer_inertia = dg::drcp_refined(k.steer_inertia);
    r.wheel_radius = dg::drcp_refined(k.wheel_radius);
    r.chassis_mass = dg::drcp_refined(k.chassis_mass);
    r.yaw_inertia = dg::drcp_refined(k.yaw_inertia);
    r.i_axle = dg::drcp_refined(k.i_axle);
    r.wheelbase = dg::drcp_refined(k.wheelbase);
    r.bbox_half = dg::drcp_refined(k.bbox_half);
    r.speed_norm = dg::drcp_refined(k.speed_norm);
    r.pi = dg::drcp_refined(3.141592653589793);
    r.ttc_max = dg::drcp_refined(k.ttc_max);
    r.road_radius = dg::drcp_refined(k.road_radius);
    r.lane_sigma = dg::drcp_refined(k.lane_sigma);
    return r;
}

struct KArgs {
    DgDims d;
    DgConsts k;
    Rcp rc;
    // engine tables
    const uint8_t* scene_blob;
    const int64_t* scene_meta;
    const int32_t* scene_of_world;
    const double* grid_offset;
    const double* mu_eff;
    const double* weather;
    const uint8_t* valid;
    const double* length;
    const double* width;
    const double* r_hull;
    const double* d_hull;
    double* state;
    uint8_t* alive;
    int8_t* reason;
    uint8_t* event_seen;
    int32_t* spawn_step;
    int32_t* step_count;
    double* start_xy;
    double* goal_xy;
    double* start_yaw;
    int32_t* error_word;
    // step io
    const void* actions;
    int32_t actions_f64;
    int32_t autoreset;
    float* obs;
    double* rewards;
    uint8_t* dones;
    uint8_t* events;
    int8_t* reason_out;
    uint8_t* alive_out;
    uint8_t* alive_pre_out;
    double* ttc_min_out;
    double* terms_out;
    double* snapshot_out;
    double* next_actions;   // fused LaneFollower output for the next tick (NULL = off)
    uint32_t* event_counts; // [W][5] episode counters, accumulated (NULL = off)
    int32_t ticks;          // control ticks per launch (persistent rollout; 1 = one step)
    int32_t ring_slots;     // obs ring: tick t writes slot (ring_start + t) % ring_slots
    int32_t ring_start;
    double pol_gain, pol_throttle;
    int32_t take_road;   // min(k_road, max_segments) = candidate-list capacity
    int32_t take_veh;    // min(k_vehicles, M)
    uint8_t* scratch;    // split mode: AgentRec[W*M], int32 world_ok[W], int32 world_step[W]
    double* drac_max;    // [W][M] running max of the per-step pairwise DRAC (NULL = off)
    uint8_t* metric_seen; // [W][M] |= goal (bit 0) / collision (bit 1) events (NULL = off)
    int32_t* index_out;   // [slot][W][M][index_stride] integer decisions (NULL = off)
    int32_t index_stride; // 3 + take_veh + take_road
    int16_t* prefix_out;  // [slot][W][M][2] non-zero obs prefix: 5 n_r, 7 n_v floats (NULL = off)
    int32_t obs_resident; // 1: obs slots keep zeros beyond prefix_out's recorded prefixes
    unsigned long long* phase_cycles; // [5] device cycles per phase, summed (NULL = off)
};

// ----------------------------------------------------------------- numpy-semantics helpers
// numpy maximum/minimum propagate NaN from either side; clip is min(max()).
// (one compare + NaN test + select; fmin/fmax on f64 expand to ~8 SASS ops)
__device__ __forceinline__ double np_max(double a, double b) { return (a != a || a > b) ? a : b; }
__device__ __forceinline__ double np_min(double a, double b) { return (a != a || a < b) ? a : b; }
// plain selects for values that cannot be NaN (or whose NaN is irrelevant)
__device__ __forceinline__ double sel_min(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double sel_clip(double x, double lo, double hi) {
    return x < lo ? lo : (x > hi ? hi : x);
}
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
    return np_min(np_max(x, lo), hi);
}
// The same with a bound that cannot be NaN (constants): one unordered compare
// (a NaN `a` still propagates) instead of two -- shorter float64 dependency chains.
__device__ __forceinline__ double np_max_k(double a, double b) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.gtu.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}" : "=d"(r) : "d"(a), "d"(b));
    return r;
}
__device__ __forceinline__ double np_min_k(double a, double b) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.ltu.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}" : "=d"(r) : "d"(a), "d"(b));
    return r;
}
__device__ __forceinline__ double np_clip_k(double x, double lo, double hi) { return np_min_k(np_max_k(x, lo), hi); }
__device__ __forceinline__ double np_sign(double x) {
    return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : (x == 0.0 ? 0.0 : x));
}
__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

__device__ __forceinline__ double4 ldg4(const double4* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ double warp_min(double v, int width = 32) {
    for (int o = width >> 1; o > 0; o >>= 1) v = sel_min(v, __shfl_xor_sync(kFull, v, o, width));
    return v;
}

__device__ __forceinline__ double warp_max_nn(double v, int width = 32) {   // non-negative values
    for (int o = width >> 1; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(kFull, v, o, width);
        v = u > v ? u : v;
    }
    return v;
}

// DRAC of the ordered pair (ego e, other n), metrics.py:33-62: d = p_n - p_e,
// u = v_n - v_e (world frame), closing = -(d.u) / max(|d|, 1e-9), clearance =
// min over the 3x3 hull-circle pairs of the centre distance - (r_e + r_n);
// closing^2 / (2 max(clearance, 1e-2)) if closing > 0 and clearance > 1e-2,
// else 0.  The caller masks dead agents and e == n.  IEEE / and sqrt (not the
// fast-path helpers): squared clearances can be arbitrarily small.  min of
// square roots == square root of the min (sqrt is correctly rounded, hence
// monotone), so one sqrt replaces nine.
__device__ __forceinline__ double pair_drac(double dx, double dy, double ux, double uy, const double* ehx,
                                            const double* ehy, const double* nhx, const double* nhy,
                                            double rsum) {
    const double dist = sqrt(dx * dx + dy * dy);
    const double closing = -(dx * ux + dy * uy) / np_max(dist, 1e-9);
    double m2 = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const double ex = ehx[a] - nhx[b], ey = ehy[a] - nhy[b];
            m2 = sel_min(m2, ex * ex + ey * ey);
        }
    const double clear = sqrt(m2) - rsum;
    return (closing > 0.0 && clear > 1e-2) ? closing * closing / (2.0 * np_max(clear, 1e-2)) : 0.0;
}

// ----------------------------------------------------------------- shared-memory layout
struct AgentSm {
    double st[DG_NUM_STATE];  // post-physics state
    double px0, py0;          // pre-physics position (progress term)
    double c, s;              // cos/sin(yaw)
    double vwx, vwy;          // world-frame velocity
    double r, d, len, wid;    // hull radius/offset, length, width
    double hx[3], hy[3];      // hull circle centres
    double gx, gy, sx, sy;    // goal, start (global)
    float f_len, f_wid, f_spd; // neighbour-row features of this agent: L/100, W/100, speed/10
    int alive, valid, reason, seen, spawn;
    // persistent rollout: the next tick's state and flags, actions, start heading
    double st_next[DG_NUM_STATE];
    double act[3];
    double start_yaw;
    int flags_next[4];
};

struct SceneView {
    double2* mid;             // [P]  segment midpoints (global after the fix-up pass)
    const double2* dir;       // [P]  unit directions
    const double* hl;         // [P]  half lengths
    const double* hw;         // [P]  half widths
    const float* type_feat;   // [P]  float32(type / type_norm), precomputed on the host
    double4* lane_seg;        // [KL] lane subset {mid x, mid y, dir x, dir y}
    const double* lane_hl;    // [KL]
    double2* edge_mid;        // [KE] edge subset midpoints
    const int32_t* edge;      // [KE] edge subset -> segment index
    // spatial index (paper_2605_08528_b200/spatial.py); flags == 0 -> full scans.
    // Header in shared memory, candidate lists in global memory (L1-cached).
    double gx0, gy0, cell, half;
    int nx, ny, words, flags;
    const int32_t* road_start;  // [nx*ny + 1]
    const uint16_t* road_list;  // segments with midpoint within `half` of the cell, ascending;
                                // bit 15 set when the segment is a road edge
    const int32_t* lane_start;  // [nx*ny + 1]
    const uint16_t* lane_list;  // lane-subset indices that can be the nearest lane, ascending
    const uint32_t* edge_bits;  // [words] bit q: segment q is a road edge
    int P, KL, KE;
};

constexpr int kFlagGrid = 1;
constexpr int kFlagLanes = 2;

__host__ __device__ __forceinline__ int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

__device__ __forceinline__ SceneView scene_view(uint8_t* base, const uint8_t* aux, int P, int KL, int KE) {
    SceneView v;
    int64_t o = 0;
    v.mid = reinterpret_cast<double2*>(base + o); o += int64_t(P) * 16;
    v.dir = reinterpret_cast<const double2*>(base + o); o += int64_t(P) * 16;
    v.hl = reinterpret_cast<const double*>(base + o); o += align16(int64_t(P) * 8);
    v.hw = reinterpret_cast<const double*>(base + o); o += align16(int64_t(P) * 8);
    v.type_feat = reinterpret_cast<const float*>(base + o); o += align16(int64_t(P) * 4);
    v.lane_seg = reinterpret_cast<double4*>(base + o); o += int64_t(KL) * 32;
    v.lane_hl = reinterpret_cast<const double*>(base + o); o += align16(int64_t(KL) * 8);
    v.edge_mid = reinterpret_cast<double2*>(base + o); o += int64_t(KE) * 16;
    v.edge = reinterpret_cast<const int32_t*>(base + o); o += align16(int64_t(KE) * 4);
    const double* hd = reinterpret_cast<const double*>(base + o);
    const int32_t* hi = reinterpret_cast<const int32_t*>(base + o + 32);
    v.gx0 = hd[0]; v.gy0 = hd[1]; v.cell = hd[2]; v.half = hd[3];
    v.nx = hi[0]; v.ny = hi[1]; v.words = hi[2]; v.flags = hi[3];
    v.road_start = reinterpret_cast<const int32_t*>(aux);
    v.road_list = reinterpret_cast<const uint16_t*>(aux + hi[4]);
    v.lane_start = reinterpret_cast<const int32_t*>(aux + hi[5]);
    v.lane_list = reinterpret_cast<const uint16_t*>(aux + hi[6]);
    v.edge_bits = reinterpret_cast<const uint32_t*>(aux + hi[7]);
    v.P = P; v.KL = KL; v.KE = KE;
    return v;
}

// ----------------------------------------------------------------- TMA bulk copy helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
// TMA bulk store shared -> global (bulk async-group completion)
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(gdst), "r"(smem_addr(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}"
        ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}

// ----------------------------------------------------------------- vehicle dynamics
struct Act {
    double thr, steer, brk;
};

// sin / cos of a steering angle (|x| <= 0.75 rad; the column clips at 1.05 theta_max):
// Taylor series in x^2 to x^17 / x^16 by fused Horner steps -- truncation below
// 1e-19, within 1 ulp of libm over the range (checked against numpy), and a
// dependency chain of 10 FMAs instead of the general sincos' range reduction on
// the substep's critical path.  Larger angles take sincos.
__device__ __forceinline__ void sincos_steer(double x, double* s, double* c) {
    if (!(fabs(x) <= 0.75)) {
        sincos(x, s, c);
        return;
    }
    const double z = x * x;
    double ps = 1.0 / 355687428096000.0;
    ps = dg::fma_rn(ps, z, -1.0 / 1307674368000.0);
    ps = dg::fma_rn(ps, z, 1.0 / 6227020800.0);
    ps = dg::fma_rn(ps, z, -1.0 / 39916800.0);
    ps = dg::fma_rn(ps, z, 1.0 / 362880.0);
    ps = dg::fma_rn(ps, z, -1.0 / 5040.0);
    ps = dg::fma_rn(ps, z, 1.0 / 120.0);
    ps = dg::fma_rn(ps, z, -1.0 / 6.0);
    double pc = 1.0 / 20922789888000.0;
    pc = dg::fma_rn(pc, z, -1.0 / 87178291200.0);
    pc = dg::fma_rn(pc, z, 1.0 / 479001600.0);
    pc = dg::fma_rn(pc, z, -1.0 / 3628800.0);
    pc = dg::fma_rn(pc, z, 1.0 / 40320.0);
    pc = dg::fma_rn(pc, z, -1.0 / 720.0);
    pc = dg::fma_rn(pc, z, 1.0 / 24.0);
    pc = dg::fma_rn(pc, z, -0.5);
    *s = dg::fma_rn(x * z, ps, x);
    *c = dg::fma_rn(z, pc, 1.0);
}

// One 120 Hz substep of the single-track model (vehicle.py:237-336), with the
// reference's expression order; x[] is the 12-field state.
__device__ __forceinline__ void substep_dynamic(double* x, const Act a, double cap, const DgConsts& k,
                                                const Rcp& rc) {
    double tau_s = np_clip_k(k.kp_steer * (k.theta_max * a.steer - x[SANG]) - k.kd_steer * x[SRATE],
                           -k.tau_steer_max, k.tau_steer_max);
    double rate = x[SRATE] + dg::ddiv_y(tau_s, k.steer_inertia, rc.steer_inertia) * k.physics_dt;
    double ang = x[SANG] + rate * k.physics_dt;
    double ang_c = np_clip_k(ang, -k.steer_limit, k.steer_limit);
    rate = (ang_c == ang) ? rate : 0.0;
    ang = ang_c;

    const double vx = x[SVX], vy = x[SVY], om = x[SOM];
    // brake torques with the wheel-sign latch (vehicle.py:182-191)
    double sf = (fabs(x[SWF]) >= 1e-4) ? np_sign(x[SWF]) : x[SBF];
    double sr = (fabs(x[SWR]) >= 1e-4) ? np_sign(x[SWR]) : x[SBR];
    double tbf = -sf * a.brk * k.tau_brake_front;
    double tbr = -sr * a.brk * k.tau_brake_rear;
    double t_front = 2.0 * (k.tau_drive_max * a.thr + tbf);
    double t_rear = 2.0 * tbr;
    double fxf0 = dg::ddiv_y(t_front, k.wheel_radius, rc.wheel_radius);
    double fxr0 = dg::ddiv_y(t_rear, k.wheel_radius, rc.wheel_radius);
    double den = np_max_k(vx, 0.5);
    const double rden = dg::drcp_refined(den);          // one reciprocal for both divisions
    double fyf0 = k.cornering_stiffness * (ang - dg::ddiv_y(vy + k.a_f * om, den, rden));
    double fyr0 = k.cornering_stiffness * dg::ddiv_y(-(vy - k.b_r * om), den, rden);

    double nf = dg::dsqrt(fxf0 * fxf0 + fyf0 * fyf0);
    double nr = dg::dsqrt(fxr0 * fxr0 + fyr0 * fyr0);
    bool satf = nf > cap, satr = nr > cap;
    double kf = satf ? dg::ddiv(cap, np_max_k(nf, 1e-12)) : 1.0;
    double kr = satr ? dg::ddiv(cap, np_max_k(nr, 1e-12)) : 1.0;
    double fxf = fxf0 * kf, fyf = fyf0 * kf;
    double fxr = fxr0 * kr, fyr = fyr0 * kr;

    double sd, cd;
    sincos_steer(ang, &sd, &cd);
    const double m = k.chassis_mass;
    double ax = dg::ddiv_y(fxf * cd - fyf * sd + fxr, m, rc.chassis_mass) + vy * om;
    double ay = dg::ddiv_y(fyf * cd + fxf * sd + fyr - k.lambda_lat * vy, m, rc.chassis_mass) - vx * om;
    double omd = dg::ddiv_y(k.a_f * (fyf * cd + fxf * sd) - k.b_r * fyr - k.lambda_yaw * om, k.yaw_inertia,
                            rc.yaw_inertia);
    double vx1 = vx + ax * k.physics_dt;
    double vy1 = vy + ay * k.physics_dt;
    double om1 = om + omd * k.physics_dt;
    if (a.brk > 0.0 && vx >= 0.0 && vx1 < 0.0) vx1 = 0.0;

    double sy, cy;
    sincos(x[SYAW], &sy, &cy);
    x[SX] = x[SX] + (vx1 * cy - vy1 * sy) * k.physics_dt;
    x[SY] = x[SY] + (vx1 * sy + vy1 * cy) * k.physics_dt;
    x[SYAW] = x[SYAW] + om1 * k.physics_dt;

    double roll_f = dg::ddiv_y((vy1 + k.a_f * om1) * sd + vx1 * cd, k.wheel_radius, rc.wheel_radius);
    double roll_r = dg::ddiv_y(vx1, k.wheel_radius, rc.wheel_radius);
    double spin_f = x[SWF] + dg::ddiv_y(t_front - fxf * k.wheel_radius, k.i_axle, rc.i_axle) * k.physics_dt;
    double spin_r = x[SWR] + dg::ddiv_y(t_rear - fxr * k.wheel_radius, k.i_axle, rc.i_axle) * k.physics_dt;
    if (a.brk > 0.0 && spin_f * sf < 0.0) spin_f = 0.0;
    if (a.brk > 0.0 && spin_r * sr < 0.0) spin_r = 0.0;
    x[SWF] = np_clip_k(satf ? spin_f : roll_f, -200.0, 200.0);
    x[SWR] = np_clip_k(satr ? spin_r : roll_r, -200.0, 200.0);
    x[SVX] = vx1;
    x[SVY] = vy1;
    x[SOM] = om1;
    x[SANG] = ang;
    x[SRATE] = rate;
    x[SBF] = sf;
    x[SBR] = sr;
}

// One 30 Hz kinematic bicycle tick (vehicle.py:208-232).
__device__ __forceinline__ void step_bicycle(double* x, const Act a, const DgConsts& k, const Rcp& rc) {
    double delta = a.steer * k.bic_steer_max;
    double v = x[SVX];
    double v1 = np_max(v + (a.thr * k.bic_a_max - a.brk * k.bic_b_max - np_sign(v) * k.bic_c_roll) * k.control_dt, 0.0);
    double yaw = x[SYAW];
    double rate = dg::ddiv_y(v1 * tan(delta), k.wheelbase, rc.wheelbase);
    double sy, cy;
    sincos(yaw, &sy, &cy);
    x[SX] = x[SX] + v1 * cy * k.control_dt;
    x[SY] = x[SY] + v1 * sy * k.control_dt;
    x[SYAW] = yaw + rate * k.control_dt;
    x[SVX] = v1;
    x[SVY] = 0.0;
    x[SOM] = rate;
    x[SANG] = delta;
    x[SRATE] = 0.0;
    x[SWF] = dg::ddiv_y(v1, k.wheel_radius, rc.wheel_radius);
    x[SWR] = dg::ddiv_y(v1, k.wheel_radius, rc.wheel_radius);
}

// ----------------------------------------------------------------- swept-circle TTC
// Minimum over the 3x3 circle pairs of the closest-approach time of agent B
// relative to ego A (observation.py:128-181).  Bit-exact restatement with one
// division per pair set: all nine pairs share a = |u|^2, and x -> fl(x / 2a)
// is monotone, so min_i fl(n_i / 2a) == fl(min_i n_i / 2a).
__device__ __forceinline__ double swept_ttc(double dx, double dy, double ux, double uy,
                                            double ce, double se, double de,
                                            double cn, double sn, double dn,
                                            double rsum, double tmax) {
    // neighbours behind the ego carry no threat (decided first: it overrides)
    if (ce * dx + se * dy < 0.0) return tmax;
    const double a = ux * ux + uy * uy;
    const bool moving = a >= 1e-12;
    // Far-pair filter: every circle pair's centre offset is p + o with
    // |o| <= de + dn, so if the closest approach of the hull centres over
    // t >= 0 stays beyond rsum + de + dn (+1e-4 m of slack over the float64
    // rounding of the exact test) no pair can hit: the result is tmax.
    {
        const double reach = rsum + de + dn + 1e-4;
        const double R2 = reach * reach;
        const double pp = dx * dx + dy * dy;
        if (moving) {
            const double pu = dx * ux + dy * uy;
            if (pu >= 0.0 ? pp > R2 : pp * a - pu * pu > R2 * a) return tmax;
        } else if (pp > R2) {
            return tmax;
        }
    }
    const double a4 = 4.0 * a;
    const double rr = rsum * rsum;
    const double offs[3] = {-1.0, 0.0, 1.0};
    bool any_overlap = false;
    double nmin = INFINITY;  // min over pairs with t_exit >= 0 of the t_enter numerator
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double oe = offs[i] * de;
        const double oec = oe * ce, oes = oe * se;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double on = offs[j] * dn;
            const double qx = dx + on * cn - oec;
            const double qy = dy + on * sn - oes;
            const double b = 2.0 * (qx * ux + qy * uy);
            const double c = qx * qx + qy * qy - rr;
            if (moving) {
                const double disc = b * b - a4 * c;
                if (disc >= 0.0) {
                    const double root = dg::dsqrt(disc);
                    if (-b + root >= 0.0) nmin = sel_min(nmin, -b - root);  // t_exit >= 0 (2a > 0)
                }
            } else if (c < 0.0) {
                any_overlap = true;
            }
        }
    }
    if (moving) return nmin < INFINITY ? sel_clip(dg::ddiv(nmin, 2.0 * a), 0.0, tmax) : tmax;
    return any_overlap ? 0.0 : tmax;
}

// ----------------------------------------------------------------- observation rows
// A row is mostly zeros (~190 of 1929 values are non-zero): the world's block
// is cleared by TMA bulk stores, then -- ordered by a barrier -- the non-zero
// features are scattered by the lanes that computed them.
// Per-agent results of the warp scans, consumed by the finalize warp.
struct ScanSm {
    double ttc_min;
    double lane_d2;
    double gap;
    int lane_k;
    int edge_hit;
    int touch;
    int pad_;
};

// ----------------------------------------------------------------- ego block / finalize
// Both launch modes share these: the ego features of one agent's row
// (observation.py:51-75) and the reward / event / termination tail of one
// agent (rewards.py:106-268, engine.py:370-406, 472-509).
// atan2(sin t, cos t) (observation.py:246-247, the neighbour heading feature):
// t itself reduced by whole turns.  Off the +-pi seam the two agree to ~1e-14
// (far below the float32 the feature is stored in); near the seam, where the
// sign of the result depends on the last bits of sin t, the exact composition
// runs instead.
__device__ __forceinline__ double wrap_angle(double t) {
    const double r = t - 6.283185307179586 * rint(t * 0.15915494309189535);
    if (fabs(r) < 3.1415) return r;
    double st, ct;
    sincos(t, &st, &ct);
    return atan2(st, ct);
}

// (sin, cos) of atan2(y, x) (observation.py:58-64): y / r, x / r; the exact
// composition where r is 0 or not finite (signed-zero quadrants).
__device__ __forceinline__ void sincos_of_bearing(double y, double x, double r, double* sh, double* ch) {
    if (r > 0.0 && r < INFINITY) {
        *sh = dg::ddiv(y, r);
        *ch = dg::ddiv(x, r);
    } else {
        sincos(atan2(y, x), sh, ch);
    }
}

__device__ __forceinline__ void write_ego(float* row, const DgConsts& k, const KArgs& A, int w, int64_t am,
                                          double px, double py, double c, double s, double vx, double vy,
                                          double gx, double gy, double* act_sm = nullptr) {
    const double gdx = gx - px, gdy = gy - py;
    const double xb = c * gdx + s * gdy;
    const double yb = -s * gdx + c * gdy;
    const double dist = dg::dsqrt(xb * xb + yb * yb);
    double sh, ch;
    sincos_of_bearing(yb, xb, dist, &sh, &ch);
    const float f2 = __double2float_rn(sh), f3 = __double2float_rn(ch);
    const float f4 = __double2float_rn(dg::ddiv_y(dist, k.bbox_half, A.rc.bbox_half));
    row[0] = __double2float_rn(dg::ddiv_y(xb, k.bbox_half, A.rc.bbox_half));
    row[1] = __double2float_rn(dg::ddiv_y(yb, k.bbox_half, A.rc.bbox_half));
    row[2] = f2;
    row[3] = f3;
    row[4] = f4;
    if (A.next_actions) {
        // LaneFollower (policies.py:21-43) on this float32 observation, fused:
        // the next tick's actions never leave the GPU
        const double sin_e = double(f2), cos_e = double(f3);
        const double dist = double(f4) * k.bbox_half;
        double steer = np_clip(A.pol_gain * sin_e, -1.0, 1.0);
        if (cos_e < 0.0) steer = sin_e >= 0.0 ? 1.0 : -1.0;
        const double thr = dist > 5.0 ? A.pol_throttle : A.pol_throttle * 0.5;
        double* act = A.next_actions + 3 * am;
        act[0] = thr;
        act[1] = steer;
        act[2] = 0.0;
        if (act_sm) {
            act_sm[0] = thr;
            act_sm[1] = steer;
            act_sm[2] = 0.0;
        }
    }
    row[5] = __double2float_rn(dg::ddiv_y(vx, k.speed_norm, A.rc.speed_norm));
    row[6] = __double2float_rn(dg::ddiv_y(vy, k.speed_norm, A.rc.speed_norm));
    if (A.d.include_weather) {
#pragma unroll
        for (int i = 0; i < 4; ++i) row[7 + i] = __double2float_rn(A.weather[4 * w + i]);
    }
}

// Output pointers of one tick (the rollout advances them by one [W][M] plane per tick).
struct TickOut {
    double* rewards;
    uint8_t* dones;
    uint8_t* events;
    int8_t* reason_out;
    uint8_t* alive_out;
    uint8_t* alive_pre_out;
    double* ttc_min_out;
    double* terms_out;
    double* snapshot_out;
};

__device__ __forceinline__ TickOut tick_out(const KArgs& A, int t) {
    const int64_t WM = int64_t(A.d.W) * A.d.M;
    TickOut o;
    o.rewards = A.rewards + t * WM;
    o.dones = A.dones + t * WM;
    o.events = A.events + t * WM * 4;
    o.reason_out = A.reason_out ? A.reason_out + t * WM : nullptr;
    o.alive_out = A.alive_out ? A.alive_out + t * WM : nullptr;
    o.alive_pre_out = A.alive_pre_out ? A.alive_pre_out + t * WM : nullptr;
    o.ttc_min_out = A.ttc_min_out ? A.ttc_min_out + t * WM : nullptr;
    o.terms_out = A.terms_out ? A.terms_out + t * WM * 7 : nullptr;
    o.snapshot_out = A.snapshot_out ? A.snapshot_out + t * WM * DG_NUM_STATE : nullptr;
    return o;
}

struct FinIn {
    const double* st;                  // post-physics state, 12 fields
    double c, s;                       // cos / sin of the post-physics yaw
    double px0, py0, gx, gy, sx, sy;   // pre-physics position, goal, start
    double lane_d2, lane_lat, lane_tx, lane_ty;  // nearest lane (d2 = inf: none)
    double ttc_min, gap;
    int edge_hit, touch, alive, valid, reason, seen, spawn;
    double start_yaw;
    bool store_global;                 // write the post-tail state to the engine arrays
    double* st_out;                    // optional: post-tail state for the next tick (shared memory)
    int* flags_out;                    // optional: alive, reason, seen, spawn after the tail
};

// What the tail decided for one agent this tick (decide_agent), consumed by
// the outputs (emit_agent): the one-hot event, reason / alive as reported
// (before an autoreset), done-or-timed-out.
struct TailRes {
    int rnow;        // 0 none, 1 goal, 2 collision, 3 crash, 4 lane_forbidden
    int reason;      // info["reason"]
    int alive_new;   // info["alive"]
    int finished;    // dones
    int park;        // done, not timed out: parked off-stage (engine.py:388-391)
};

// Events and termination of one agent this tick (rewards.py:206-268 sparse
// part, engine.py:370-393 tail): the reported reason / alive and done flag.
__device__ __forceinline__ TailRes tail_events(const KArgs& A, const FinIn& F, int step_now, int* seen_new) {
            const DgConsts& k = A.k;
            const double px = F.st[SX], py = F.st[SY];
            const double vx = F.st[SVX], vy = F.st[SVY];
            const double tgx = F.gx - px, tgy = F.gy - py;
            const double speed = dg::dsqrt(vx * vx + vy * vy);
            const bool alive = F.alive;
            const bool goal = dg::dsqrt(tgx * tgx + tgy * tgy) <= k.goal_radius;
            const double sxd = px - F.sx, syd = py - F.sy;
            const bool bad = !(finite(px) && finite(py) && finite(vx) && finite(vy));
            const bool crash = dg::dsqrt(sxd * sxd + syd * syd) > k.crash_drift_limit || bad ||
                               speed > k.crash_speed_limit;
            const bool coll = F.touch && step_now - F.spawn >= A.d.collision_warmup;
            const int seen = F.seen;
            const bool e_goal = goal && alive && !(seen & 1);
            const bool e_coll = coll && alive && !(seen & 2);
            const bool e_crash = crash && alive && !(seen & 4);
            const bool e_lf = F.edge_hit && alive && !(seen & 8);
            const int rnow = e_goal ? 1 : (e_crash ? 3 : (e_lf ? 4 : (e_coll ? 2 : 0)));
            *seen_new = seen | (rnow == 0 ? 0 : 1 << (rnow == 1 ? 0 : rnow == 2 ? 1 : rnow == 3 ? 2 : 3));
            int reason = F.reason;
            bool done = false;
            if (!A.d.invincible) {
                done = rnow != 0;
                if (done && reason == 0) reason = rnow;
            }
            const int step_new = step_now + 1;
            const bool timeout = step_new >= A.d.episode_len && alive;
            const bool finished = done || timeout;
            if (timeout && reason == 0) reason = 5;
            TailRes R;
            R.rnow = rnow;
            R.reason = reason;
            R.alive_new = alive && !finished;
            R.finished = finished;
            R.park = done && !timeout;
            return R;
}

// The post-tail state of one agent (engine.py:388-393 park, 599-619 autoreset
// teleport) -> st_out / flags_out and, when store_global, the engine arrays;
// returns the agent's contribution to the episode counters: bits 0..3 the
// one-hot event (goal, collision, crash, lane_forbidden), bit 4 alive before
// the tick, kBitFinished.
__device__ __forceinline__ unsigned tail_state(const KArgs& A, int w, int m, const FinIn& F, const TailRes& R,
                                               int seen_new, int step_now, double ox, double oy) {
            const DgConsts& k = A.k;
            const int WM = A.d.W * A.d.M;
            const int64_t am = int64_t(w) * A.d.M + m;
            const bool park = R.park;
            int alive_new = R.alive_new, reason = R.reason;
            double x[DG_NUM_STATE];
#pragma unroll
            for (int f = 0; f < DG_NUM_STATE; ++f) x[f] = F.st[f];
            if (park) {
#pragma unroll
                for (int f = 0; f < DG_NUM_STATE; ++f) x[f] = (f == SBF || f == SBR) ? 1.0 : 0.0;
                x[SX] = ox + k.offstage_x;
                x[SY] = oy;
            }
            int spawn = F.spawn;
            if (A.autoreset && R.finished && F.valid) {
#pragma unroll
                for (int f = 0; f < DG_NUM_STATE; ++f) x[f] = (f == SBF || f == SBR) ? 1.0 : 0.0;
                x[SX] = F.sx;
                x[SY] = F.sy;
                x[SYAW] = F.start_yaw;
                alive_new = 1;
                reason = 0;
                spawn = step_now + 1;
                seen_new = 0;
            }
            if (F.store_global) {
#pragma unroll
                for (int f = 0; f < DG_NUM_STATE; ++f) A.state[int64_t(f) * WM + am] = x[f];
                A.alive[am] = uint8_t(alive_new);
                A.reason[am] = int8_t(reason);
                A.event_seen[am] = uint8_t(seen_new);
                A.spawn_step[am] = spawn;
            }
            if (F.st_out) {
#pragma unroll
                for (int f = 0; f < DG_NUM_STATE; ++f) F.st_out[f] = x[f];
                F.flags_out[0] = alive_new;
                F.flags_out[1] = reason;
                F.flags_out[2] = seen_new;
                F.flags_out[3] = spawn;
            }
            const int rnow = R.rnow;
            return (rnow == 0 ? 0u : 1u << (rnow == 1 ? 0 : rnow == 2 ? 1 : rnow == 3 ? 2 : 3)) |
                   (F.alive ? 16u : 0u) | (R.finished ? kBitFinished : 0u);
}

// decide (events + post-tail state) now, emit later (the pipelined fused tail)
__device__ __forceinline__ unsigned decide_agent(const KArgs& A, int w, int m, const FinIn& F, int step_now,
                                                 double ox, double oy, TailRes* R) {
    int seen_new;
    *R = tail_events(A, F, step_now, &seen_new);
    return tail_state(A, w, m, F, *R, seen_new, step_now, ox, oy);
}

// The dense reward terms (rewards.py:106-204), the sparse reward of the decided
// event, and every per-tick output of one agent (StepOutput, engine.py:397-406).
__device__ __forceinline__ void emit_agent(const KArgs& A, const TickOut& O, int w, int m, const FinIn& F,
                                           const TailRes& R) {
            const DgConsts& k = A.k;
            const int WM = A.d.W * A.d.M;
            const int64_t am = int64_t(w) * A.d.M + m;
            const double px = F.st[SX], py = F.st[SY];
            const double vx = F.st[SVX], vy = F.st[SVY];
            const double dist = dg::dsqrt(F.lane_d2);
            const bool has_lane = finite(dist);
            const double lat = has_lane ? F.lane_lat : 0.0;
            double tx = has_lane ? F.lane_tx : 0.0, ty = has_lane ? F.lane_ty : 0.0;
            const double tgx = F.gx - px, tgy = F.gy - py;
            const double flip = (tx * tgx + ty * tgy >= 0.0) ? 1.0 : -1.0;
            tx = tx * flip;
            ty = ty * flip;
            double progress = np_clip_k((px - F.px0) * tx + (py - F.py0) * ty,
                                      -k.progress_clamp, k.progress_clamp) * k.progress_weight;
            // cos(yaw - atan2(ty, tx)) (rewards.py:127-128) as the dot product of the
            // heading with the unit lane tangent: same value to ~1e-16, no atan2 / cos
            // on the tail's critical path (yaw NaN -> NaN, as numpy)
            const double align = np_max(0.0, F.c * tx + F.s * ty);
            const double ls = dg::ddiv_y(lat, k.lane_sigma, A.rc.lane_sigma);
            const double quality = exp(-(ls * ls)) * (k.lane_heading_base + k.lane_heading_weight * align);
            const double lane_t = has_lane ? k.lane_weight * quality : 0.0;
            progress = has_lane ? progress : 0.0;
            const double offroad = (has_lane && (fabs(lat) > k.offroad_lat_limit || dist > k.offroad_dist_limit))
                                       ? -k.offroad_weight : 0.0;
            const double speed = dg::dsqrt(vx * vx + vy * vy);
            const double idle = speed < k.idle_speed ? -k.idle_weight : 0.0;
            const double ttc_v = -np_min_k(dg::ddiv(k.ttc_vehicle_alpha, np_max_k(F.ttc_min, k.ttc_floor)),
                                           k.ttc_vehicle_pmax);
            const double tau = F.gap < INFINITY ? dg::ddiv(F.gap, np_max_k(vx, 0.1)) : F.gap / np_max_k(vx, 0.1);
            const double ttc_e = finite(tau) ? -np_min_k(dg::ddiv(k.ttc_edge_alpha, np_max_k(tau, k.ttc_floor)), k.ttc_edge_pmax)
                                             : 0.0;
            const double total = progress + lane_t + offroad + idle + ttc_v + ttc_e;
            const int rnow = R.rnow;
            const double sparse = rnow == 1 ? k.goal_weight
                                : rnow == 2 ? -k.collision_weight
                                : rnow == 3 ? -k.crash_weight
                                : rnow == 4 ? -k.lane_forbidden_weight : 0.0;
            const bool alive = F.alive;
            const double reward = alive ? total + sparse : 0.0;

            if (A.metric_seen && (rnow == 1 || rnow == 2)) A.metric_seen[am] |= uint8_t(rnow == 1 ? 1 : 2);
            O.rewards[am] = reward;
            O.dones[am] = uint8_t(R.finished);
            reinterpret_cast<uint32_t*>(O.events)[am] =
                uint32_t(rnow == 1) | (uint32_t(rnow == 2) << 8) | (uint32_t(rnow == 3) << 16) |
                (uint32_t(rnow == 4) << 24);
            if (O.reason_out) O.reason_out[am] = int8_t(R.reason);
            if (O.alive_out) O.alive_out[am] = uint8_t(R.alive_new);
            if (O.alive_pre_out) O.alive_pre_out[am] = uint8_t(alive);
            if (O.ttc_min_out) O.ttc_min_out[am] = F.ttc_min;
            if (O.terms_out) {
                const double t7[7] = {progress, lane_t, offroad, idle, ttc_v, ttc_e, total};
#pragma unroll
                for (int i = 0; i < 7; ++i) O.terms_out[int64_t(i) * WM + am] = alive ? t7[i] : 0.0;
            }
            if (O.snapshot_out) {
#pragma unroll
                for (int f = 0; f < DG_NUM_STATE; ++f) O.snapshot_out[int64_t(f) * WM + am] = F.st[f];
            }
}

// decide + emit in one pass (the split kernels and the unpipelined fused tail)
__device__ __forceinline__ unsigned finalize_agent(const KArgs& A, const TickOut& O, int w, int m, const FinIn& F,
                                                   int step_now, double ox, double oy) {
    int seen_new;
    const TailRes R = tail_events(A, F, step_now, &seen_new);
    emit_agent(A, O, w, m, F, R);
    return tail_state(A, w, m, F, R, seen_new, step_now, ox, oy);
}

// Episode counters [W][5] (goal, collision, crash, lane_forbidden, alive
// agent-ticks), accumulated over ticks: warp-reduced, one add per counter.
__device__ __forceinline__ void count_events(const KArgs& A, int w, unsigned bits, unsigned active_mask, bool leader,
                                             bool atomic) {
    if (!A.event_counts) return;
    unsigned c[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) c[i] = __popc(__ballot_sync(active_mask, (bits >> i) & 1u));
    if (leader) {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if (!c[i]) continue;
            if (atomic) atomicAdd(A.event_counts + 5 * w + i, c[i]);
            else A.event_counts[5 * w + i] += c[i];
        }
    }
}

// ----------------------------------------------------------------- optional phase timers
// Built with -DDG_PHASE_TIMERS: every CTA records clock64() at its phase
// boundaries (slot 0 start .. 7 end) plus the per-warp end of phase 2.
#ifdef DG_PHASE_TIMERS
__device__ long long g_phase_clock[65536][40];
#define PHASE_MARK(i) do { if (threadIdx.x == 0 && blockIdx.x < 65536) g_phase_clock[blockIdx.x][i] = clock64(); } while (0)
#define WARP_MARK(i) do { if ((threadIdx.x & 31) == 0 && blockIdx.x < 65536) g_phase_clock[blockIdx.x][8 + (threadIdx.x >> 5)] = clock64(); } while (0)
#define LANE0_MARK(i) do { if (threadIdx.x == 0 && blockIdx.x < 65536) g_phase_clock[blockIdx.x][i] = clock64(); } while (0)
__device__ __forceinline__ long long gtimer() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
#define GT_MARK(i) do { if (threadIdx.x == 0 && blockIdx.x < 65536) g_phase_clock[blockIdx.x][i] = gtimer(); } while (0)
#define W1_MARK(i) do { if (threadIdx.x == 32 && blockIdx.x < 65536) g_phase_clock[blockIdx.x][i] = clock64(); } while (0)
#else
#define GT_MARK(i) do { } while (0)
#define W1_MARK(i) do { } while (0)
#define LANE0_MARK(i) do { } while (0)
#define PHASE_MARK(i) do { } while (0)
#define WARP_MARK(i) do { } while (0)
#endif

// Built with -DDG_TICK_TIMERS: per-CTA clock64 sums over every tick of a
// (multi-tick) launch -- slots 0..4 the phases of thread 0's tick (action
// check, phase 1, phase 2 incl. its barrier, tail, closing barrier), 8 + w the
// scan time of warp w, 30 / 31 the physics warp's ego block / physics.
#ifdef DG_TICK_TIMERS
// per-CTA cycle sums in shared memory (one writer per slot), copied out once at
// the end of the launch: no global read-modify-write inside the timed ticks
__device__ long long g_tick_acc[65536][48];
#define TT_DECL __shared__ long long s_tt[48]; \
    if (threadIdx.x < 48) s_tt[threadIdx.x] = 0; \
    __syncthreads(); \
    long long tt_last = clock64(), tt_w = 0; (void)tt_w
#define TT_ACC(i) do { if (threadIdx.x == 0) { const long long n_ = clock64(); s_tt[i] += n_ - tt_last; tt_last = n_; } } while (0)
#define TT_WSTART() do { if ((threadIdx.x & 31) == 0) tt_w = clock64(); } while (0)
#define TT_WACC(i) do { if ((threadIdx.x & 31) == 0) { const long long n_ = clock64(); s_tt[i] += n_ - tt_w; tt_w = n_; } } while (0)
#define TT_FLUSH() do { __syncthreads(); if (threadIdx.x < 48) g_tick_acc[blockIdx.x][threadIdx.x] = s_tt[threadIdx.x]; } while (0)
#else
#define TT_FLUSH() do { } while (0)
#define TT_DECL do { } while (0)
#define TT_ACC(i) do { } while (0)
#define TT_WSTART() do { } while (0)
#define TT_WACC(i) do { } while (0)
#endif

// ---- per-phase device cycles (DgStepIO.phase_cycles, the reference's
// phase_seconds: action, physics, observation, reward_termination, reset).
// Lane 0 of every warp adds the cycles it spends in each phase to a shared
// counter; one global add per phase at the end of the launch.  Off (one
// predicated branch per mark) when the pointer is NULL.
enum { PH_ACTION = 0, PH_PHYSICS, PH_OBSERVATION, PH_REWARD, PH_RESET };
#define PH_START() do { if (ph_on && (threadIdx.x & 31) == 0) ph_t = clock64(); } while (0)
#define PH_ADD(i) do { if (ph_on && (threadIdx.x & 31) == 0) { const long long n_ = clock64(); \
    atomicAdd(&s_ph[i], (unsigned long long)(n_ - ph_t)); ph_t = n_; } } while (0)

// The raw (unclipped) actions of tick t for agent am: the fused policy's
// shared-memory record when `fed` is given, else the caller's [T][W][M][3] array.
__device__ __forceinline__ void load_actions(const KArgs& A, int t, int64_t am, const double* fed, double* raw) {
    if (fed) {
        raw[0] = fed[0]; raw[1] = fed[1]; raw[2] = fed[2];
        return;
    }
    const int64_t ab = int64_t(t) * A.d.W * A.d.M * 3 + am * 3;
    if (A.actions_f64) {
        const double* a = reinterpret_cast<const double*>(A.actions);
        raw[0] = a[ab]; raw[1] = a[ab + 1]; raw[2] = a[ab + 2];
    } else {
        const float* a = reinterpret_cast<const float*>(A.actions);
        raw[0] = a[ab]; raw[1] = a[ab + 1]; raw[2] = a[ab + 2];
    }
}

// Physics of one agent for one control tick (decode + decimation substeps,
// engine.py:410-421 with the alive mask) from state x0, and the derived
// per-tick record the scans read (heading cos/sin, world velocity, hull
// centres, speed feature).  run = false leaves the state as it is.
__device__ __forceinline__ void agent_physics(const KArgs& A, int w, AgentSm& S, const double* x0, int alive,
                                              const double* raw, bool run) {
    const DgConsts& k = A.k;
    double x[DG_NUM_STATE];
#pragma unroll
    for (int f = 0; f < DG_NUM_STATE; ++f) x[f] = x0[f];
    S.px0 = x[SX];
    S.py0 = x[SY];
    if (alive && x[SX] != -12345.678) LANE0_MARK(25);  // after the state loads landed
    if (run) {
        Act act;
        act.thr = np_clip(raw[0], 0.0, 1.0);
        act.steer = np_clip(raw[1], -1.0, 1.0);
        act.brk = np_clip(raw[2], 0.0, 1.0);
        if (A.d.dynamic) {
            const double cap = A.mu_eff[w] * k.f_z;
            for (int i = 0; i < A.d.decimation; ++i) {
                substep_dynamic(x, act, cap, k, A.rc);
#ifdef DG_PHASE_TIMERS
                if (i < 4 && x[SX] != -12345.678) LANE0_MARK(28 + i);
#endif
            }
        } else {
            step_bicycle(x, act, k, A.rc);
        }
    }
    if (x[SX] != -12345.678) LANE0_MARK(26);          // after the substeps
#pragma unroll
    for (int f = 0; f < DG_NUM_STATE; ++f) S.st[f] = x[f];
    double s_, c_;
    sincos(x[SYAW], &s_, &c_);
    S.c = c_;
    S.s = s_;
    S.vwx = x[SVX] * c_ - x[SVY] * s_;
    S.vwy = x[SVX] * s_ + x[SVY] * c_;
    S.f_spd = __double2float_rn(dg::ddiv_y(dg::dsqrt(x[SVX] * x[SVX] + x[SVY] * x[SVY]), k.speed_norm, A.rc.speed_norm));
    const double offs[3] = {-1.0, 0.0, 1.0};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double o = offs[i] * S.d;
        S.hx[i] = x[SX] + o * c_;
        S.hy[i] = x[SY] + o * s_;
    }
    S.alive = alive;
    LANE0_MARK(27);
}

// Zero n floats at p with a group of gsz (>= 4) lanes, li = lane in the group:
// scalar head up to 16-byte alignment, float4 body, scalar tail.
__device__ __forceinline__ void zero_span(float* p, int n, int li, int gsz) {
    if (n <= 0) return;
    int head = int((16u - unsigned(reinterpret_cast<uintptr_t>(p) & 15u)) & 15u) >> 2;
    head = head < n ? head : n;
    if (li < head) p[li] = 0.0f;
    float4* q = reinterpret_cast<float4*>(p + head);
    const int n4 = (n - head) >> 2;
    for (int i = li; i < n4; i += gsz) q[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int done = head + 4 * n4;
    if (li < n - done) p[done + li] = 0.0f;
}

// Zero n floats of observation rows at base (one warp): TMA bulk stores from
// the zeroed shared buffer for the 16-byte-aligned body (the lanes issue them
// and, with wait, wait for their completion; else every lane of the warp must
// call bulk_commit_and_wait later), plain stores for the unaligned head / tail.
__device__ __forceinline__ void zero_obs_block(float* base, int64_t n, const float4* zero_sm, int lane,
                                               bool wait = true) {
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(base);
    const uintptr_t b1 = b0 + uintptr_t(n) * 4;
    const uintptr_t a0 = (b0 + 15) & ~uintptr_t(15), a1 = b1 & ~uintptr_t(15);
    if (a0 < a1) {
        for (uintptr_t p = b0 + 4 * lane; p < a0; p += 128) *reinterpret_cast<float*>(p) = 0.0f;
        for (uintptr_t p = a1 + 4 * lane; p < b1; p += 128) *reinterpret_cast<float*>(p) = 0.0f;
        // every lane issues its share of the chunks (one bulk group per lane)
        asm volatile("fence.proxy.async.global;" ::: "memory");   // after earlier generic writes
        for (uintptr_t p = a0 + uintptr_t(lane) * kZeroChunk; p < a1; p += 32 * uintptr_t(kZeroChunk)) {
            const uintptr_t nb = a1 - p < uintptr_t(kZeroChunk) ? a1 - p : uintptr_t(kZeroChunk);
            bulk_store(reinterpret_cast<void*>(p), zero_sm, uint32_t(nb));
        }
        if (wait) bulk_commit_and_wait();
        else asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    } else {
        for (uintptr_t p = b0 + 4 * lane; p < b1; p += 128) *reinterpret_cast<float*>(p) = 0.0f;
    }
}

// FinIn of an agent from its tick record and scan results; with lanes, the
// nearest-lane terms from the scene's lane table (emit_agent needs them,
// decide_agent does not).  Flags default to the record's.
__device__ __forceinline__ FinIn fin_in(const AgentSm& S, const ScanSm& R, const SceneView& G, bool lanes) {
    FinIn F;
    F.st = S.st;
    F.c = S.c;
    F.s = S.s;
    F.px0 = S.px0; F.py0 = S.py0; F.gx = S.gx; F.gy = S.gy; F.sx = S.sx; F.sy = S.sy;
    F.lane_d2 = R.lane_d2;
    F.lane_lat = 0.0; F.lane_tx = 0.0; F.lane_ty = 0.0;
    if (lanes && R.lane_d2 < INFINITY) {
        const double4 l4 = G.lane_seg[R.lane_k];
        const double ex = S.st[SX] - l4.x, ey = S.st[SY] - l4.y;
        F.lane_tx = l4.z;
        F.lane_ty = l4.w;
        F.lane_lat = l4.z * ey - l4.w * ex;
    }
    F.ttc_min = R.ttc_min; F.gap = R.gap;
    F.edge_hit = R.edge_hit; F.touch = R.touch;
    F.alive = S.alive; F.valid = S.valid;
    F.reason = S.reason; F.seen = S.seen; F.spawn = S.spawn;
    F.start_yaw = S.start_yaw;
    F.store_global = false;
    F.st_out = nullptr;
    F.flags_out = nullptr;
    return F;
}

// Which phase-2 work units a scan warp takes: 2a units = ego pairs (egos 2u,
// 2u + 1), 2b units = groups of `apw` agents.  Default: both kinds strided over
// the warps (every warp one of each at 8 warps).  kSpec (7 scan warps beside
// the physics warp): the 2b units go two per warp to the first warps, the 2a
// units are split evenly over the rest -- measured costs ~7k / ~5k cycles per
// unit, so 16 agents on 7 warps finish in max(2 x 7k, 3 x 5k) instead of the
// 19k a strided 7-warp split would take.
struct ScanSchedule {
    int a_lo, a_hi, a_step;   // 2a units
    int b_lo, b_hi, b_step;   // 2b units
};

template <bool kSpec>
__device__ __forceinline__ ScanSchedule scan_schedule(int M, int apw, int warp, int nwarps) {
    ScanSchedule r;
    const int PA = (M + 1) / 2, PB = (M + apw - 1) / apw;
    if (!kSpec) {
        r.a_lo = warp; r.a_hi = PA; r.a_step = nwarps;
        r.b_lo = warp; r.b_hi = PB; r.b_step = nwarps;
        return r;
    }
    r.a_step = r.b_step = 1;
    int nb = (PB + 1) / 2;
    nb = nb < nwarps ? nb : nwarps;
    const int na = nwarps - nb;
    const int pb = (PB + nb - 1) / nb;
    r.b_lo = warp < nb ? warp * pb : 0;
    r.b_hi = warp < nb ? min(PB, r.b_lo + pb) : 0;
    if (na > 0) {
        const int pa = (PA + na - 1) / na;
        r.a_lo = warp >= nb ? (warp - nb) * pa : 0;
        r.a_hi = warp >= nb ? min(PA, r.a_lo + pa) : 0;
    } else {
        r.a_lo = 0;
        r.a_hi = warp == 0 ? PA : 0;
    }
    return r;
}

// ----------------------------------------------------------------- the fused step kernel
// kGeoGlobal: the world's geometry is a per-world blob already moved by the grid
// offset, read in place from global memory (L1 / L2) -- scenes too large for
// shared memory (DgDims.geometry_global); otherwise the scene blob is staged in
// shared memory by TMA and offset there.
// kPhase: the per-phase cycle counters are compiled in (DgStepIO.phase_cycles;
// instantiated for the engine's default shapes, launched only when requested --
// they cost the plain variants 2-3 % in registers even when off)
template <bool kStep, int kThreads, int kMinBlocks, bool kSpec, bool kGeoGlobal, bool kPhase = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
world_step_kernel(const KArgs A) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int w = blockIdx.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // kSpec: the last warp is the physics warp (pw); the scans run on the others
    const int nwarps = (blockDim.x >> 5) - (kSpec ? 1 : 0);
    const int pw = nwarps;
    const int M = A.d.M;
    const int WM = A.d.W * M;
    const int D = A.d.obs_dim;
    const DgConsts& k = A.k;
    TT_DECL;
    __shared__ unsigned long long s_ph[5];
    const bool ph_on = kPhase && A.phase_cycles != nullptr;
    long long ph_t = 0;
    if (ph_on && tid < 5) s_ph[tid] = 0;

    // ---- shared memory carve-up: three agent tables (kSpec: tick t is read from
    //      table t & 1 while the physics warp writes tick t + 1 into the other, and
    //      table 2 takes tick t + 1 of agents teleported back to their start); the
    //      rollout carry (st_next, flags_next, act) lives in table 0
    uint8_t* geo = smem;
    AgentSm* const ag_home = reinterpret_cast<AgentSm*>(smem + (kGeoGlobal ? 0 : align16(A.d.max_scene_bytes)));
    AgentSm* const ag_rst = ag_home + 2 * kMaxAgents;
    AgentSm* ag = ag_home;
    // scan results: two tables (kSpec: tick t's scans write table t & 1 while the
    // physics warp emits tick t - 1's outputs from the other); tail decisions
    ScanSm* const sc_base = reinterpret_cast<ScanSm*>(ag_home + 3 * kMaxAgents);
    TailRes* const tail_sm = reinterpret_cast<TailRes*>(sc_base + 2 * kMaxAgents);
    uint64_t* bar = reinterpret_cast<uint64_t*>(tail_sm + kMaxAgents);
    uint16_t* cand_sm = reinterpret_cast<uint16_t*>(bar + 2);   // [M][take_road]
    float4* zero_sm = reinterpret_cast<float4*>(
        smem + align16(reinterpret_cast<uint8_t*>(cand_sm + kMaxAgents * A.take_road) - smem));  // [kZeroChunk/16]
    for (int i = tid; i < kZeroChunk / 16; i += blockDim.x) zero_sm[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    // resident ring: this world's prefix record of every slot, cached for the launch
    // (the global record is still written every tick)
    int16_t* const pfx_sm = reinterpret_cast<int16_t*>(zero_sm + kZeroChunk / 16);   // [kPfxSlots][16][2]
    const bool pfx_cached = kStep && A.obs_resident && A.ring_slots <= kPfxSlots;
    if (pfx_cached)
        for (int i = tid; i < A.ring_slots * M * 2; i += blockDim.x) {
            const int sl = i / (2 * M), r = i % (2 * M);
            pfx_sm[(sl * kMaxAgents + r / 2) * 2 + (r & 1)] =
                A.prefix_out[(int64_t(sl) * A.d.W * M + int64_t(w) * M + r / 2) * 2 + (r & 1)];
        }
    // pairs phase: each ego's neighbour order of the previous tick (rank of agent
    // j, agent at rank r) and whether it is set
    __shared__ int8_t s_rank[kMaxAgents][kMaxAgents];
    __shared__ int8_t s_ord[kMaxAgents][kMaxAgents];
    __shared__ int8_t s_rok[kMaxAgents];
    if (tid < kMaxAgents) s_rok[tid] = 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    __shared__ int s_bad;
    const int T = kStep ? (A.ticks > 0 ? A.ticks : 1) : 1;
    const int64_t act_tick = int64_t(WM) * 3;      // actions of tick t at A.actions + t * act_tick
    const bool feedback = kStep && T > 1 && A.next_actions != nullptr;   // fused policy drives ticks >= 1

    // ---- geometry: one bulk async copy of the world's scene blob (TMA engine),
    //      once per launch; with ticks > 1 it serves the whole rollout
    const int scene = A.scene_of_world[w];
    const int64_t* meta = A.scene_meta + 8 * scene;
    const double ox = A.grid_offset[2 * w], oy = A.grid_offset[2 * w + 1];

    // ---- tick-0 action scan (the reference rejects before mutating anything)
    GT_MARK(32);
    PHASE_MARK(0);
    int step_now = 0;
    PH_START();
    if constexpr (kStep) {
        if (tid == 0) s_bad = DG_NO_ERROR;
        __syncthreads();
        if (tid < 3 * M) {
            const int64_t flat = int64_t(w) * M * 3 + tid;
            const double v = A.actions_f64 ? reinterpret_cast<const double*>(A.actions)[flat]
                                           : double(reinterpret_cast<const float*>(A.actions)[flat]);
            if (!finite(v)) atomicMin(&s_bad, int(flat));
        }
        __syncthreads();
        if (s_bad != DG_NO_ERROR) {
            if (tid == 0) atomicMin(A.error_word, s_bad);
            return;
        }
        step_now = A.step_count[w];
        PH_ADD(PH_ACTION);
    }
    if (!kGeoGlobal && tid == 0) {
        mbar_init(bar, 1);
        bulk_load(geo, A.scene_blob + meta[0], uint32_t(meta[1]), bar);
    }

    // ---- per-agent tables and the initial state -> shared memory (once)
    if (warp == 0 && lane < M) {
        const int m = lane;
        const int64_t am = int64_t(w) * M + m;
        AgentSm& S = ag[m];
#pragma unroll
        for (int f = 0; f < DG_NUM_STATE; ++f) S.st_next[f] = A.state[int64_t(f) * WM + am];
        S.flags_next[0] = A.alive[am];
        S.flags_next[1] = A.reason[am];
        S.flags_next[2] = A.event_seen[am];
        S.flags_next[3] = A.spawn_step[am];
        S.r = A.r_hull[am];
        S.d = A.d_hull[am];
        S.len = A.length[am];
        S.wid = A.width[am];
        S.f_len = __double2float_rn(dg::ddiv(S.len, k.bbox_half));
        S.f_wid = __double2float_rn(dg::ddiv(S.wid, k.bbox_half));
        S.gx = A.goal_xy[2 * am];
        S.gy = A.goal_xy[2 * am + 1];
        S.sx = A.start_xy[2 * am];
        S.sy = A.start_xy[2 * am + 1];
        S.start_yaw = A.start_yaw[am];
        S.valid = A.valid[am];
        if constexpr (kSpec) {
            for (int tb = 1; tb < 3; ++tb) {
                AgentSm& S1 = ag_home[tb * kMaxAgents + m];
                S1.r = S.r; S1.d = S.d; S1.len = S.len; S1.wid = S.wid; S1.f_len = S.f_len; S1.f_wid = S.f_wid;
                S1.gx = S.gx; S1.gy = S.gy; S1.sx = S.sx; S1.sy = S.sy; S1.start_yaw = S.start_yaw;
                S1.valid = S.valid;
            }
        }
    }
    SceneView G;
    bool zero_early = false;   // kSpec physics warp: the next slot's clear is in flight
    for (int t = 0; t < T; ++t) {
        if constexpr (kSpec) ag = ag_home + (t & 1) * kMaxAgents;
        AgentSm* const agn = ag_home + ((t + 1) & 1) * kMaxAgents;   // kSpec: tick t + 1
        (void)agn;
        ScanSm* const sc = sc_base + (kSpec ? (t & 1) * kMaxAgents : 0);
        const int slot = A.ring_slots > 0 ? (A.ring_start + t) % A.ring_slots : t;
        // kSpec pipeline: the outputs of tick t - 1 (decided at its end) are
        // emitted by the physics warp while tick t's scans run
        auto emit_prev = [&]() {
            const int tp = t - 1;
            if (lane < M) {
                const int sp = A.ring_slots > 0 ? (A.ring_start + tp) % A.ring_slots : tp;
                const FinIn F = fin_in(ag_home[(tp & 1) * kMaxAgents + lane], sc_base[(tp & 1) * kMaxAgents + lane],
                                       G, true);
                emit_agent(A, tick_out(A, sp), w, lane, F, tail_sm[lane]);
            }
        };
        float* obs_w = A.obs + (int64_t(slot) * WM + int64_t(w) * M) * D;
        int32_t* ix_w = A.index_out ? A.index_out + (int64_t(slot) * WM + int64_t(w) * M) * A.index_stride
                                    : nullptr;
        const TickOut O = tick_out(A, slot);
        if (kStep && t > 0) {
            // every tick gets the same rejection as a separate step call (s_bad was
            // reset at the end of the previous tick, before its closing barrier;
            // kSpec: the physics warp checked this tick's actions during the
            // previous tick's scans, two barriers ago)
            if (!kSpec && tid < 3 * M) {
                const int64_t flat = t * act_tick + int64_t(w) * M * 3 + tid;
                const double v = feedback ? ag_home[tid / 3].act[tid % 3]
                               : A.actions_f64 ? reinterpret_cast<const double*>(A.actions)[flat]
                                               : double(reinterpret_cast<const float*>(A.actions)[flat]);
                if (!finite(v)) atomicMin(&s_bad, int(flat));
            }
            if (!kSpec) __syncthreads();
            if (s_bad != DG_NO_ERROR) {
                // ticks 0..t-1 stand (as t separate step calls would leave them)
                if (kSpec && warp == 0) emit_prev();
                if (warp == 0 && lane < M) {
                    const int64_t am = int64_t(w) * M + lane;
                    const AgentSm& S = ag_home[lane];
#pragma unroll
                    for (int f = 0; f < DG_NUM_STATE; ++f) A.state[int64_t(f) * WM + am] = S.st_next[f];
                    A.alive[am] = uint8_t(S.flags_next[0]);
                    A.reason[am] = int8_t(S.flags_next[1]);
                    A.event_seen[am] = uint8_t(S.flags_next[2]);
                    A.spawn_step[am] = S.flags_next[3];
                }
                if (tid == 0) {
                    atomicMin(A.error_word, s_bad);
                    A.step_count[w] = step_now + t;
                }
                return;
            }
        }
        TT_ACC(0);

        PHASE_MARK(1);
        // ---- phase 1: warp 0, lane m: agent m physics (SIMT across agents).  kSpec:
        //      only tick 0 -- later ticks were computed ahead by the physics warp
        if ((!kSpec || t == 0) && warp == 0 && lane < M) {
            const int m = lane;
            const int64_t am = int64_t(w) * M + m;
            AgentSm& S = ag[m];
            const AgentSm& H = ag_home[m];
            S.reason = H.flags_next[1];
            S.seen = H.flags_next[2];
            S.spawn = H.flags_next[3];
            double raw[3] = {0.0, 0.0, 0.0};
            PH_START();
            if (kStep && H.flags_next[0]) load_actions(A, t, am, t > 0 && feedback ? H.act : nullptr, raw);
            agent_physics(A, w, S, H.st_next, H.flags_next[0], raw, kStep && H.flags_next[0]);
            PH_ADD(PH_PHYSICS);
        }
        // the zero background of the world's obs block: TMA bulk stores from a
        // zeroed shared buffer, issued by one thread of a warp that is idle
        // during the physics; unaligned head/tail floats by plain stores
        if ((!kSpec || t == 0) && !A.obs_resident && warp == (nwarps > 1 ? 1 : 0)) {
            PH_START();
            zero_obs_block(obs_w, int64_t(M) * D, zero_sm, lane);
            PH_ADD(PH_OBSERVATION);
        }

        if (warp == 0) PHASE_MARK(2);
        __syncthreads();  // agent table + zero rows done, mbarrier init visible
        PHASE_MARK(3);
        if (kGeoGlobal && t == 0) {
            G = scene_view(const_cast<uint8_t*>(A.scene_blob + meta[0]), A.scene_blob + meta[5], int(meta[2]),
                           int(meta[3]), int(meta[4]));
        } else if (t == 0) {
            mbar_wait(bar, 0);
            // the view reads the index header from the copied blob: only after the wait
            G = scene_view(geo, A.scene_blob + meta[5], int(meta[2]), int(meta[3]), int(meta[4]));
            // scene-local midpoints -> global, exactly midpoints + grid offset
            for (int i = tid; i < G.P; i += blockDim.x) {
                double2 m2 = G.mid[i];
                m2.x = m2.x + ox;
                m2.y = m2.y + oy;
                G.mid[i] = m2;
            }
            for (int i = tid; i < G.KL; i += blockDim.x) {
                double4 l4 = G.lane_seg[i];
                l4.x = l4.x + ox;
                l4.y = l4.y + oy;
                G.lane_seg[i] = l4;
            }
            for (int i = tid; i < G.KE; i += blockDim.x) {
                double2 e2 = G.edge_mid[i];
                e2.x = e2.x + ox;
                e2.y = e2.y + oy;
                G.edge_mid[i] = e2;
            }
            __syncthreads();
        }

        PHASE_MARK(4);
        TT_ACC(1);
        TT_WSTART();
        if (kSpec && warp == pw) {
            // ---- the physics warp, concurrently with the scans of tick t: lanes m < 16
            //      write the ego block of tick t (+ the fused policy's action for t + 1),
            //      check tick t + 1's actions and run its physics from this tick's
            //      post-physics state, assuming the tail leaves the agent alone (true
            //      unless it finishes); lanes 16 + m run the same physics from agent m's
            //      spawn state, the tick-(t + 1) state if the tail teleports it back
            //      (autoreset).  finalize takes that, or re-derives a parked agent.
            // the next tick's zero background: TMA bulk stores issued now, completed
            // before the tick's closing barrier -- they stream out under the scans
            // and the tail (a slot shared by consecutive ticks is cleared in the tail)
            PH_START();
            if (kStep && t > 0) {
                emit_prev();
                __syncwarp();
                PH_ADD(PH_REWARD);
            }
            const int slot1 = A.ring_slots > 0 ? (A.ring_start + t + 1) % A.ring_slots : t + 1;
            zero_early = t + 1 < T && slot1 != slot && !A.obs_resident;
#ifdef DG_EXP_NOZERO
            zero_early = false;
#endif
            if (zero_early)
                zero_obs_block(A.obs + (int64_t(slot1) * WM + int64_t(w) * M) * D, int64_t(M) * D, zero_sm, lane,
                               false);
            TT_WACC(29);
            const int m = lane & 15;
            const bool rst = lane >= 16;
            AgentSm& S = ag[m < M ? m : 0];
            AgentSm& H = ag_home[m < M ? m : 0];
            const int64_t am = int64_t(w) * M + m;
            if (!rst && m < M)
                write_ego(obs_w + int64_t(m) * D, k, A, w, am, S.st[SX], S.st[SY], S.c, S.s, S.st[SVX], S.st[SVY],
                          S.gx, S.gy, feedback ? H.act : nullptr);
            PH_ADD(PH_OBSERVATION);
            TT_WACC(30);
            __syncwarp();
            if (kStep && t + 1 < T && m < M) {
                double raw[3];
                load_actions(A, t + 1, am, feedback ? H.act : nullptr, raw);
                if (!rst) {
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        if (!finite(raw[j])) atomicMin(&s_bad, int((t + 1) * act_tick + am * 3 + j));
                }
                PH_ADD(PH_ACTION);
                const bool go = !rst || (A.autoreset && S.valid);
                double x0[DG_NUM_STATE];
#pragma unroll
                for (int f = 0; f < DG_NUM_STATE; ++f) x0[f] = rst ? ((f == SBF || f == SBR) ? 1.0 : 0.0) : S.st[f];
                if (rst) {
                    x0[SX] = S.sx;
                    x0[SY] = S.sy;
                    x0[SYAW] = S.start_yaw;
                }
                const int alive = rst ? 1 : S.alive;
                if (go) agent_physics(A, w, rst ? ag_rst[m] : agn[m], x0, alive, raw, alive != 0);
                PH_ADD(PH_PHYSICS);
            }
            TT_WACC(31);
            if (zero_early) bulk_commit_and_wait();   // the next slot's clear, before the scans of t + 1
        } else {
        // ---- phase 2a: agent pairs.  kPL lanes per ego agent, each lane owns the other
        //      agents j = jl + kPL * u (u < 16 / kPL): 16 lanes x 1 at 8 warps per world,
        //      8 lanes x 2 at 4 warps (four egos per warp in one pass).  Stable distance
        //      rank, swept-circle TTC, neighbour rows, hull contact, optional DRAC.
        PH_START();
        const int road0 = A.d.ego_dim;
        const int veh0 = A.d.ego_dim + 5 * A.d.k_road;
        const ScanSchedule sched = scan_schedule<kSpec>(M, kThreads <= 128 ? 4 : 2, warp, nwarps);
        {
            constexpr int kPL = 16;                           // lanes per ego (8 measured slower at 4 warps)
            constexpr int kOPL = kMaxAgents / kPL;            // other agents per lane
            constexpr int kEPW = 32 / kPL;                    // egos per warp
            const int grp = lane / kPL, jl = lane % kPL;
            const unsigned gmask = ((1u << kPL) - 1u) << (kPL * grp);
            for (int u = sched.a_lo; u < sched.a_hi; u += sched.a_step) {
                const int i = kEPW * u + grp;
                const bool ego_ok = i < M;
                const int ii = ego_ok ? i : 0;
                const AgentSm& S = ag[ii];
                const double px = S.st[SX], py = S.st[SY], c = S.c, s = S.s;
                double key[kOPL], ndx[kOPL], ndy[kOPL];
#pragma unroll
                for (int u = 0; u < kOPL; ++u) {
                    const int j = jl + kPL * u;
                    key[u] = INFINITY;
                    ndx[u] = 0.0;
                    ndy[u] = 0.0;
                    if (ego_ok && j < M) {
                        const AgentSm& N = ag[j];
                        ndx[u] = N.st[SX] - px;
                        ndy[u] = N.st[SY] - py;
                        const double dist = dg::dsqrt(ndx[u] * ndx[u] + ndy[u] * ndy[u]);
                        key[u] = (N.alive && j != ii) ? dist : INFINITY;
                    }
                }
                int rank[kOPL];
#pragma unroll
                for (int u = 0; u < kOPL; ++u) rank[u] = 0;
                // The previous tick's order is reused when it still sorts this tick's
                // keys: every agent's key against its predecessor's in that order (one
                // shuffle) -- a sorted permutation is unique, so the ranks are the stable
                // argsort's.  Otherwise (or at a launch's first tick) the full count.
                bool full = true;
                if constexpr (kOPL == 1) {
                    const bool have = ego_ok && jl < M && s_rok[ii];
                    const int r0 = have ? int(s_rank[ii][jl]) : 0;
                    const int pj = have && r0 > 0 ? int(s_ord[ii][r0 - 1]) : jl;
                    const double kp = __shfl_sync(kFull, key[0], pj, kPL);
                    const bool ok = !ego_ok || jl >= M || (have && (r0 == 0 || kp < key[0] ||
                                                                    (kp == key[0] && pj < jl)));
                    full = !__all_sync(kFull, ok);
                    rank[0] = r0;
                }
                if (full) {
#pragma unroll
                for (int u = 0; u < kOPL; ++u) rank[u] = 0;
#pragma unroll
                for (int v = 0; v < kOPL; ++v)
                    for (int sl = 0; sl < kPL; ++sl) {
                        const int t = sl + kPL * v;
                        const double kt = __shfl_sync(kFull, key[v], sl, kPL);
                        if (t < M) {
#pragma unroll
                            for (int u = 0; u < kOPL; ++u) {
                                const int j = jl + kPL * u;
                                rank[u] += (kt < key[u]) || (kt == key[u] && t < j);
                            }
                        }
                    }
                    if constexpr (kOPL == 1) {
                        if (ego_ok && jl < M) {
                            s_rank[ii][jl] = int8_t(rank[0]);
                            s_ord[ii][rank[0]] = int8_t(jl);
                        }
                        __syncwarp();
                        if (ego_ok && jl == 0) s_rok[ii] = 1;
                    }
                }
                TT_WACC(32 + (warp & 7) % 3);     // 2a sub-timers: key + rank
                double ttc = k.ttc_max;
                bool touch = false;
                double dr = 0.0;
                int n_valid = 0;
#pragma unroll
                for (int u = 0; u < kOPL; ++u) {
                    const int j = jl + kPL * u;
                    const bool nvalid = ego_ok && j < M && finite(key[u]) && rank[u] < A.take_veh;
                    n_valid += nvalid;
                    if (nvalid && ix_w) ix_w[int64_t(ii) * A.index_stride + 3 + rank[u]] = j;
                    if (nvalid) {
                        const AgentSm& N = ag[j];
                        const double tj = swept_ttc(ndx[u], ndy[u], N.vwx - S.vwx, N.vwy - S.vwy, c, s, S.d, N.c,
                                                    N.s, N.d, S.r + N.r, k.ttc_max);
                        ttc = sel_min(ttc, tj);
                        const double wrap = wrap_angle(N.st[SYAW] - S.st[SYAW]);
                        float* o = obs_w + int64_t(ii) * D + veh0 + 7 * rank[u];
                        o[0] = __double2float_rn(dg::ddiv_y(c * ndx[u] + s * ndy[u], k.bbox_half, A.rc.bbox_half));
                        o[1] = __double2float_rn(dg::ddiv_y(-s * ndx[u] + c * ndy[u], k.bbox_half, A.rc.bbox_half));
                        o[2] = N.f_len;
                        o[3] = N.f_wid;
                        o[4] = __double2float_rn(dg::ddiv_y(wrap, 3.141592653589793, A.rc.pi));
                        o[5] = N.f_spd;
                        o[6] = __double2float_rn(dg::ddiv_y(tj, k.ttc_max, A.rc.ttc_max));
                    }
                    // hull contact; centres sit within d of the position, so a pair
                    // farther apart than r_a + r_b + d_a + d_b (+1e-4 m) cannot touch
                    if (kStep && ego_ok && j < M && j != ii && S.alive && ag[j].alive &&
                        key[u] <= S.r + ag[j].r + S.d + ag[j].d + 1e-4) {
                        const AgentSm& N = ag[j];
                        const double rs = S.r + N.r;
                        const double rs2 = rs * rs;
    #pragma unroll
                        for (int a = 0; a < 3; ++a)
    #pragma unroll
                            for (int b = 0; b < 3; ++b) {
                                const double ex = S.hx[a] - N.hx[b], ey = S.hy[a] - N.hy[b];
                                touch |= ex * ex + ey * ey < rs2;
                            }
                    }
                    if (kStep && A.drac_max && ego_ok && j < M && j != ii && S.alive && ag[j].alive) {
                        // episode safety metric on the post-physics state, agents alive before the tick
                        const AgentSm& N = ag[j];
                        const double d1 = pair_drac(ndx[u], ndy[u], N.vwx - S.vwx, N.vwy - S.vwy, S.hx, S.hy,
                                                    N.hx, N.hy, S.r + N.r);
                        dr = d1 > dr ? d1 : dr;
                    }
                }
                TT_WACC(35 + (warp & 7) % 3);     // TTC, rows, contact
                ttc = warp_min(ttc, kPL);
                touch = (__ballot_sync(kFull, touch) & gmask) != 0;
                if (ix_w || A.prefix_out) {
                    if constexpr (kOPL == 1) {
                        n_valid = __popc(__ballot_sync(kFull, n_valid != 0) & gmask);   // one vote, no chain
                    } else {
                        for (int o = kPL / 2; o > 0; o >>= 1) n_valid += __shfl_xor_sync(kFull, n_valid, o, kPL);
                    }
                    if (ix_w && ego_ok && jl == 0) ix_w[int64_t(ii) * A.index_stride + 2] = n_valid;
                    if (A.prefix_out && ego_ok) {
                        int16_t* pre = A.prefix_out + (int64_t(slot) * WM + int64_t(w) * M + ii) * 2 + 1;
                        // resident obs: the row holds zeros past its previous prefix; clear
                        // only the rows the previous tick of this slot had beyond n_valid
                        int16_t* const pc = pfx_sm + (slot * kMaxAgents + ii) * 2 + 1;
                        const int old_v = !A.obs_resident ? 0
                                          : min(int(pfx_cached ? *pc : *pre), 7 * A.d.k_vehicles);
                        __syncwarp(gmask);
                        if (jl == 0) {
                            *pre = int16_t(7 * n_valid);
                            if (pfx_cached) *pc = int16_t(7 * n_valid);
                        }
                        if (old_v > 7 * n_valid)
                            zero_span(obs_w + int64_t(ii) * D + veh0 + 7 * n_valid, old_v - 7 * n_valid, jl, kPL);
                    }
                }

                if (kStep && A.drac_max) {
                    dr = warp_max_nn(dr, kPL);
                    if (ego_ok && jl == 0) {
                        double* p = A.drac_max + int64_t(w) * M + ii;
                        const double prev = *p;
                        *p = dr > prev ? dr : prev;
                    }
                }
                if (ego_ok && jl == 0) {
                    sc[ii].ttc_min = ttc;
                    sc[ii].touch = touch;
                    if (!kStep && A.ttc_min_out) A.ttc_min_out[int64_t(w) * M + ii] = ttc;
                }
                TT_WACC(38 + (warp & 7) % 3);     // reductions, prefix, sc
            }
        }

        W1_MARK(34);
        TT_WACC(20 + warp);
        PH_ADD(PH_OBSERVATION);
        // ---- phase 2b: each lane group scans the scene for one agent -- a warp takes
        //      kAPW consecutive agents (16 lanes x 2 at 8 warps per world, 8 lanes x 4 at
        //      4 warps), so the agents' dependent load / reduction chains overlap in one
        //      instruction stream.  Lists are walked in kGL-entry chunks (every group
        //      iterates to the longest list, predicated); collectives are full-warp with
        //      per-group masks, reductions are kGL-lane shuffles.
        constexpr int kGL = kThreads <= 128 ? 8 : 16;       // lanes per agent
        constexpr int kAPW = 32 / kGL;                      // agents per warp
        constexpr unsigned kGMask = (1u << kGL) - 1u;
        for (int pr = sched.b_lo; pr < sched.b_hi; pr += sched.b_step) {
            const int half = lane / kGL, hl = lane % kGL;
            const unsigned hshift = unsigned(kGL) * unsigned(half);
            const int m = kAPW * pr + half;
            const bool act = m < M;                     // a short last group leaves lanes idle
            const AgentSm& S = ag[act ? m : kAPW * pr];
            float* row = obs_w + int64_t(act ? m : kAPW * pr) * D;
            const double px = S.st[SX], py = S.st[SY];
            const double c = S.c, s = S.s;
            const bool rewards_needed = kStep && act && S.alive;   // dead agents: rewards/events masked
            const double r2 = S.r * S.r;
            bool edge_hit = false;

            // (a) road context: exact d2 <= r^2 over the candidate superset, ordered
            //     compaction into shared memory; edge boxes tested on the same pass
            uint16_t* cand = cand_sm + (act ? m : kAPW * pr) * A.take_road;
            int count = 0;
            auto visit = [&](int q, bool in, bool edge_q) {
                bool hit = false;
                if (in) {
                    const double2 m2 = G.mid[q];
                    const double dx = m2.x - px, dy = m2.y - py;
                    const double d2 = dx * dx + dy * dy;
                    hit = d2 <= k.road_radius_sq;
                    if (rewards_needed && edge_q) {
                        const double hl_ = G.hl[q], hw_ = G.hw[q];
                        const double reach = S.r + S.d + hl_ + hw_ + 1e-6;
                        if (d2 <= reach * reach) {
                            const double2 u2 = G.dir[q];
    #pragma unroll
                            for (int i = 0; i < 3; ++i) {
                                const double qx = S.hx[i] - m2.x, qy = S.hy[i] - m2.y;
                                const double along = qx * u2.x + qy * u2.y;
                                const double lat = u2.x * qy - u2.y * qx;
                                const double du = along - sel_clip(along, -hl_, hl_);
                                const double dv = lat - sel_clip(lat, -hw_, hw_);
                                edge_hit |= du * du + dv * dv < r2;
                            }
                        }
                    }
                }
                const unsigned bal = (__ballot_sync(kFull, hit) >> hshift) & kGMask;
                if (hit) {
                    const int slot = count + __popc(bal & ((1u << hl) - 1u));
                    if (slot < A.take_road) cand[slot] = uint16_t(q);
                }
                count += __popc(bal);
            };
            const bool use_grid = (G.flags & kFlagGrid) != 0;
            // the agent's grid cell (scene-local coordinates); -1 off the grid
            int cell_id = -1;
            if (G.flags && act) {
                const double inv = 1.0 / G.cell;
                const double fx = floor((px - ox - G.gx0) * inv), fy = floor((py - oy - G.gy0) * inv);
                if (fx >= 0.0 && fy >= 0.0 && fx < double(G.nx) && fy < double(G.ny)) cell_id = int(fy) * G.nx + int(fx);
            }
            // the cell's list bounds and the first lane candidates, loaded together up
            // front (independent of the road pass; consumed by the lane pass below)
            const int lcell = (G.flags & kFlagLanes) ? cell_id : -1;
            int lo = 0, hi = 0, lb0 = 0, lb1 = 0, lfirst = 0;
            if (use_grid && cell_id >= 0) {
                lo = __ldg(G.road_start + cell_id);
                hi = __ldg(G.road_start + cell_id + 1);
            }
            if (lcell >= 0) {
                lb0 = __ldg(G.lane_start + lcell);
                lb1 = __ldg(G.lane_start + lcell + 1);
                if (lb0 + hl < lb1) lfirst = __ldg(G.lane_list + lb0 + hl);
            }
            if (use_grid) {
                // the cell's superset list (ascending) -> exact predicates, index order;
                // off the grid nothing is within the road radius or an edge box
                int nt_max = (hi - lo + kGL - 1) / kGL;
                for (int o = kGL; o < 32; o <<= 1) nt_max = max(nt_max, __shfl_xor_sync(kFull, nt_max, o));
                for (int it = 0; it < nt_max; ++it) {
                    const int i = lo + kGL * it + hl;
                    const bool in = i < hi;
                    const int e = in ? int(__ldg(G.road_list + i)) : 0;
                    visit(e & 0x7fff, in, (e >> 15) != 0);
                }
            } else {
                for (int p0 = 0; p0 < G.P; p0 += kGL) visit(p0 + hl, act && p0 + hl < G.P, false);
            }
            const int ncand = count < A.take_road ? count : A.take_road;
            __syncwarp();
            int32_t* ix_m = ix_w ? ix_w + int64_t(act ? m : kAPW * pr) * A.index_stride : nullptr;
            if (act) {
                if (ix_m && hl == 0) ix_m[1] = ncand;
                if (A.prefix_out) {
                    int16_t* pre = A.prefix_out + (int64_t(slot) * WM + int64_t(w) * M + m) * 2;
                    // resident obs: the previous prefix (0x7fff: slot written elsewhere -> all)
                    int16_t* const pc = pfx_sm + (slot * kMaxAgents + m) * 2;
                    const int old_r = !A.obs_resident ? 0 : min(int(pfx_cached ? *pc : *pre), 5 * A.d.k_road);
                    __syncwarp(kGMask << hshift);
                    if (hl == 0) {
                        *pre = int16_t(5 * ncand);
                        if (pfx_cached) *pc = int16_t(5 * ncand);
                    }
                    if (old_r > 5 * ncand) zero_span(row + road0 + 5 * ncand, old_r - 5 * ncand, hl, kGL);
                }
                for (int slot = hl; slot < ncand; slot += kGL) {
                    const int q = cand[slot];
                    if (ix_m) ix_m[3 + A.take_veh + slot] = q;
                    const double2 m2 = G.mid[q], u2 = G.dir[q];
                    const double dx = m2.x - px, dy = m2.y - py;
                    const double ux = u2.x, uy = u2.y;
                    float* o = row + road0 + 5 * slot;
                    o[0] = __double2float_rn(dg::ddiv_y(c * dx + s * dy, k.road_radius, A.rc.road_radius));
                    o[1] = __double2float_rn(dg::ddiv_y(-s * dx + c * dy, k.road_radius, A.rc.road_radius));
                    o[2] = G.type_feat[q];
                    o[3] = __double2float_rn(c * ux + s * uy);
                    o[4] = __double2float_rn(-s * ux + c * uy);
                }
            }
            // both agents dead (or absent): no rewards / events -> skip the rest
            if (!__any_sync(kFull, rewards_needed)) {
                if (ix_m && act && hl == 0) ix_m[0] = -1;
                if (kStep && act && hl == 0) {
                    ScanSm& R = sc[m];
                    R.lane_d2 = INFINITY;
                    R.lane_k = 0;
                    R.gap = INFINITY;
                    R.edge_hit = 0;
                }
                continue;
            }
            // (b) first road edge ahead over every edge (xb in (0, edge_range]); the
            //     edge boxes when the grid could not take them
            double gap = INFINITY;
    #pragma unroll 2
            for (int kk = hl; kk < G.KE; kk += kGL) {
                const double2 m2 = G.edge_mid[kk];
                const double ex = m2.x - px, ey = m2.y - py;
                const double xb = c * ex + s * ey;
                if (xb > 0.0 && xb <= k.edge_range && xb < gap) gap = xb;
                if (!use_grid && rewards_needed) {
                    const int q = G.edge[kk];
                    const double2 u2 = G.dir[q];
                    const double hl_ = G.hl[q], hw_ = G.hw[q];
                    const double reach = S.r + S.d + hl_ + hw_ + 1e-6;
                    if (ex * ex + ey * ey <= reach * reach) {
    #pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            const double qx = S.hx[i] - m2.x, qy = S.hy[i] - m2.y;
                            const double along = qx * u2.x + qy * u2.y;
                            const double lat = u2.x * qy - u2.y * qx;
                            const double du = along - sel_clip(along, -hl_, hl_);
                            const double dv = lat - sel_clip(lat, -hw_, hw_);
                            edge_hit |= du * du + dv * dv < r2;
                        }
                    }
                }
            }
            gap = warp_min(gap, kGL);
            edge_hit = ((__ballot_sync(kFull, edge_hit) >> hshift) & kGMask) != 0;

            // (c) nearest lane: argmin of point-to-segment d2, lowest index on ties,
            //     over the cell's candidate list when the agent is inside the grid
            double best = INFINITY;
            int best_k = 0x7fffffff;
            auto lane_test = [&](int kk) {
                const double4 l4 = G.lane_seg[kk];
                const double ex = px - l4.x, ey = py - l4.y;
                const double along = ex * l4.z + ey * l4.w;
                const double lat = l4.z * ey - l4.w * ex;
                const double t = fabs(along) - G.lane_hl[kk];
                const double over = t > 0.0 ? t : 0.0;   // NaN along -> NaN lat, d2 NaN either way
                const double d2 = over * over + lat * lat;
                if (d2 < best) { best = d2; best_k = kk; }
            };
            if (lcell >= 0) {
                if (lb0 + hl < lb1) lane_test(lfirst);
                for (int i = lb0 + kGL + hl; i < lb1; i += kGL) lane_test(__ldg(G.lane_list + i));
            } else if (act) {
                for (int kk = hl; kk < G.KL; kk += kGL) lane_test(kk);
            }
            for (int o = kGL / 2; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(kFull, best, o, kGL);
                const int ok = __shfl_xor_sync(kFull, best_k, o, kGL);
                if (ob < best || (ob == best && ok < best_k)) { best = ob; best_k = ok; }
            }
            if (ix_m && act && hl == 0) ix_m[0] = rewards_needed && best < INFINITY ? best_k : -1;
            if (kStep && act && hl == 0) {
                ScanSm& R = sc[m];
                if (rewards_needed) {
                    R.lane_d2 = best;
                    R.lane_k = best_k;
                    R.gap = gap;
                    R.edge_hit = edge_hit;
                } else {
                    R.lane_d2 = INFINITY;
                    R.lane_k = 0;
                    R.gap = INFINITY;
                    R.edge_hit = 0;
                }
            }
        }
        TT_WACC(8 + warp);
        PH_ADD(PH_OBSERVATION);
        }   // phase 2 (kSpec: the scan warps)
        WARP_MARK(0);
        __syncthreads();
        PHASE_MARK(5);
        TT_ACC(2);

        // ---- phase 3: one lane per agent (SIMT across the world's agents):
        //      warp 0 -> rewards, events, termination, state for the next tick;
        //      warp 1 (or warp 0 afterwards) -> the ego block (+ fused policy)
        const int ego_warp = nwarps > 1 ? 1 : 0;
        if (!kSpec && warp == ego_warp && lane < M) {
            AgentSm& S = ag[lane];
            PH_START();
            write_ego(obs_w + int64_t(lane) * D, k, A, w, int64_t(w) * M + lane, S.st[SX], S.st[SY], S.c, S.s,
                      S.st[SVX], S.st[SVY], S.gx, S.gy, feedback ? S.act : nullptr);
            PH_ADD(PH_OBSERVATION);
        }
        if constexpr (kStep) {
            if (warp == 0 && lane < M) {
                // kSpec: decide now (events, termination, the state tick t + 1 starts
                // from), emit the outputs during tick t + 1's scans -- or here after
                // the last tick; otherwise both here
                const int m = lane;
                AgentSm& S = ag[m];
                AgentSm& H = ag_home[m];
                FinIn F = fin_in(S, sc[m], G, !kSpec || t + 1 == T);
                if (kSpec) {
                    F.reason = H.flags_next[1];
                    F.seen = H.flags_next[2];
                    F.spawn = H.flags_next[3];
                }
                F.store_global = t + 1 == T;
                F.st_out = H.st_next;
                F.flags_out = H.flags_next;
                PH_START();
                TT_ACC(5);
                unsigned bits;
                if constexpr (kSpec) {
                    bits = decide_agent(A, w, m, F, step_now + t, ox, oy, &tail_sm[m]);
                    if (t + 1 == T) emit_agent(A, O, w, m, F, tail_sm[m]);
                } else {
                    bits = finalize_agent(A, O, w, m, F, step_now + t, ox, oy);
                }
                TT_ACC(6);
                count_events(A, w, bits, __activemask(), lane == 0, false);
                TT_ACC(7);
                PH_ADD(PH_REWARD);
#ifdef DG_EXP_NOFIX
                if (false) {
#else
                if (kSpec && t + 1 < T && (bits & kBitFinished)) {
#endif
                    // the tail moved the agent: teleported back to its start -> the
                    // physics warp's spawn-state branch; parked / timed out -> dead,
                    // no physics, the record re-derived from the post-tail state
                    AgentSm& N1 = agn[m];
                    if (H.flags_next[0]) {
                        const AgentSm& R1 = ag_rst[m];
#pragma unroll
                        for (int f = 0; f < DG_NUM_STATE; ++f) N1.st[f] = R1.st[f];
                        N1.px0 = R1.px0; N1.py0 = R1.py0; N1.c = R1.c; N1.s = R1.s;
                        N1.vwx = R1.vwx; N1.vwy = R1.vwy; N1.f_spd = R1.f_spd;
#pragma unroll
                        for (int i = 0; i < 3; ++i) { N1.hx[i] = R1.hx[i]; N1.hy[i] = R1.hy[i]; }
                        N1.alive = 1;
                    } else {
                        const double none[3] = {0.0, 0.0, 0.0};
                        agent_physics(A, w, N1, H.st_next, 0, none, false);
                    }
                }
                PH_ADD(PH_RESET);
            }

            if (kSpec && warp == pw && t + 1 < T && !zero_early && !A.obs_resident) {
#ifndef DG_EXP_NOZERO
                // consecutive ticks share the slot: clear it after this tick's scans
                const int slot1 = A.ring_slots > 0 ? (A.ring_start + t + 1) % A.ring_slots : t + 1;
                zero_obs_block(A.obs + (int64_t(slot1) * WM + int64_t(w) * M) * D, int64_t(M) * D, zero_sm, lane);
#endif
            }
            if (tid == 0) A.step_count[w] = step_now + t + 1;
            PHASE_MARK(6);
            GT_MARK(33);
            TT_ACC(3);
        }
        if (!kSpec && kStep && tid == 0) s_bad = DG_NO_ERROR;   // for the next tick's action check
        if (t + 1 < T) __syncthreads();   // next tick reads st_next / act written above
        TT_ACC(4);
    }
    TT_FLUSH();
    if (ph_on) {
        __syncthreads();
        if (tid < 5 && s_ph[tid]) atomicAdd(A.phase_cycles + tid, s_ph[tid]);
    }
}

// ----------------------------------------------------------------- split launch mode
// Two kernels per tick, chained with programmatic dependent launch (PDL):
//   K1 world_physics_kernel  one warp per world, lane m = agent m: action
//      scan, decode, 4 substeps (SIMT across agents), derived per-agent
//      record -> global scratch, post-physics state -> state[], step counter
//   K2 agent_obs_kernel      one warp per agent, a few agents of one world
//      per CTA: clears its obs rows with TMA bulk stores *before* waiting on
//      K1 (griddepcontrol.wait), then pairs / road / edges / lane scans,
//      the ego block and the agent's own reward / termination tail.
// Every SM gets many independent agent warps, so the scans of one agent
// hide the latency chains of another; the physics chain costs one short
// kernel instead of a CTA-wide barrier stall.
struct __align__(16) AgentRec {
    double x, y, yaw, vx, vy, c, s, vwx, vwy, r, d;
    double hx[3], hy[3];
    float f_len, f_wid, f_spd;
    int alive;
};

// scratch: AgentRec rec[W*M] | int32 world_ok[W], int32 world_step[W] | double2 prev_pos[W*M]
__host__ __device__ __forceinline__ int64_t split_off_world(int W, int M) {
    return align16(int64_t(sizeof(AgentRec)) * W * M);
}
__host__ __device__ __forceinline__ int64_t split_off_prev(int W, int M) {
    return split_off_world(W, M) + align16(int64_t(8) * W);
}
__host__ __device__ __forceinline__ size_t split_scratch_bytes(int W, int M) {
    return size_t(split_off_prev(W, M) + align16(int64_t(16) * W * M));
}

template <bool kStep>
__global__ void __launch_bounds__(32) world_physics_kernel(const KArgs A) {
    const int w = blockIdx.x;
    const int lane = threadIdx.x;
    const int M = A.d.M;
    const int WM = A.d.W * M;
    const DgConsts& k = A.k;
    AgentRec* rec = reinterpret_cast<AgentRec*>(A.scratch);
    int32_t* world_ok = reinterpret_cast<int32_t*>(A.scratch + split_off_world(A.d.W, M));
    int32_t* world_step = world_ok + A.d.W;
    double2* prev = reinterpret_cast<double2*>(A.scratch + split_off_prev(A.d.W, M));
    // let the dependent agent kernel start its independent prologue now
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if constexpr (kStep) {
        int bad = DG_NO_ERROR;
        for (int i = lane; i < 3 * M; i += 32) {
            const int64_t flat = int64_t(w) * M * 3 + i;
            const double v = A.actions_f64 ? reinterpret_cast<const double*>(A.actions)[flat]
                                           : double(reinterpret_cast<const float*>(A.actions)[flat]);
            if (!finite(v) && int(flat) < bad) bad = int(flat);
        }
        for (int o = 16; o > 0; o >>= 1) {
            const int ob = __shfl_xor_sync(kFull, bad, o);
            bad = ob < bad ? ob : bad;
        }
        if (bad != DG_NO_ERROR) {   // the reference rejects before mutating anything
            if (lane == 0) {
                atomicMin(A.error_word, bad);
                world_ok[w] = 0;
            }
            return;
        }
        if (lane == 0) {
            const int step_now = A.step_count[w];
            world_ok[w] = 1;
            world_step[w] = step_now;
            A.step_count[w] = step_now + 1;
        }
    }
    if (lane >= M) return;
    const int m = lane;
    const int64_t am = int64_t(w) * M + m;
    double x[DG_NUM_STATE];
#pragma unroll
    for (int f = 0; f < DG_NUM_STATE; ++f) x[f] = A.state[int64_t(f) * WM + am];
    const int alive = A.alive[am];
    const double px0 = x[SX], py0 = x[SY];
    if (kStep && alive) {
        const int64_t ab = am * 3;
        double raw0, raw1, raw2;
        if (A.actions_f64) {
            const double* a = reinterpret_cast<const double*>(A.actions);
            raw0 = a[ab]; raw1 = a[ab + 1]; raw2 = a[ab + 2];
        } else {
            const float* a = reinterpret_cast<const float*>(A.actions);
            raw0 = a[ab]; raw1 = a[ab + 1]; raw2 = a[ab + 2];
        }
        Act act;
        act.thr = np_clip(raw0, 0.0, 1.0);
        act.steer = np_clip(raw1, -1.0, 1.0);
        act.brk = np_clip(raw2, 0.0, 1.0);
        if (A.d.dynamic) {
            const double cap = A.mu_eff[w] * k.f_z;
            for (int i = 0; i < A.d.decimation; ++i) substep_dynamic(x, act, cap, k, A.rc);
        } else {
            step_bicycle(x, act, k, A.rc);
        }
        // the post-physics state (the info snapshot; the tail parks from here)
#pragma unroll
        for (int f = 0; f < DG_NUM_STATE; ++f) A.state[int64_t(f) * WM + am] = x[f];
    }
    AgentRec R;
    double s_, c_;
    sincos(x[SYAW], &s_, &c_);
    R.x = x[SX]; R.y = x[SY]; R.yaw = x[SYAW]; R.vx = x[SVX]; R.vy = x[SVY];
    R.c = c_; R.s = s_;
    R.vwx = x[SVX] * c_ - x[SVY] * s_;
    R.vwy = x[SVX] * s_ + x[SVY] * c_;
    R.r = A.r_hull[am];
    R.d = A.d_hull[am];
    const double offs[3] = {-1.0, 0.0, 1.0};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double o = offs[i] * R.d;
        R.hx[i] = x[SX] + o * c_;
        R.hy[i] = x[SY] + o * s_;
    }
    R.f_len = __double2float_rn(dg::ddiv(A.length[am], k.bbox_half));
    R.f_wid = __double2float_rn(dg::ddiv(A.width[am], k.bbox_half));
    R.f_spd = __double2float_rn(dg::ddiv(dg::dsqrt(x[SVX] * x[SVX] + x[SVY] * x[SVY]), k.speed_norm));
    R.alive = alive;
    rec[am] = R;
    prev[am] = make_double2(px0, py0);
}

template <bool kStep, int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) agent_obs_kernel(const KArgs A) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int apc = blockDim.x >> 5;              // agents (warps) per CTA
    const int M = A.d.M;
    const int groups = (M + apc - 1) / apc;
    const int w = blockIdx.x / groups;
    const int m0 = (blockIdx.x % groups) * apc;
    const int mc = M - m0 < apc ? M - m0 : apc;   // agents in this CTA
    const int WM = A.d.W * M;
    const int D = A.d.obs_dim;
    const DgConsts& k = A.k;
    const AgentRec* rec = reinterpret_cast<const AgentRec*>(A.scratch);
    const int32_t* world_ok = reinterpret_cast<const int32_t*>(A.scratch + split_off_world(A.d.W, M));
    const int32_t* world_step = world_ok + A.d.W;
    const double2* prev = reinterpret_cast<const double2*>(A.scratch + split_off_prev(A.d.W, M));

    AgentRec* ag = reinterpret_cast<AgentRec*>(smem);                          // [M]
    uint16_t* cand_sm = reinterpret_cast<uint16_t*>(ag + kMaxAgents);        // [apc][take_road]
    float4* zero_sm = reinterpret_cast<float4*>(
        smem + align16(reinterpret_cast<uint8_t*>(cand_sm + apc * A.take_road) - smem));

    // ---- prologue, independent of K1: clear this CTA's obs rows (TMA bulk stores);
    //      one tick per launch, written to ring slot ring_start (header contract)
    const int slot = A.ring_start;
    float* rows = A.obs + (int64_t(slot) * WM + int64_t(w) * M + m0) * D;
    for (int i = tid; i < kZeroChunk / 16; i += blockDim.x) zero_sm[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        const uintptr_t b0 = reinterpret_cast<uintptr_t>(rows);
        const uintptr_t b1 = b0 + uintptr_t(mc) * D * 4;
        const uintptr_t a0 = (b0 + 15) & ~uintptr_t(15), a1 = b1 & ~uintptr_t(15);
        if (a0 < a1) {
            for (uintptr_t p = b0 + 4 * lane; p < a0; p += 128) *reinterpret_cast<float*>(p) = 0.0f;
            for (uintptr_t p = a1 + 4 * lane; p < b1; p += 128) *reinterpret_cast<float*>(p) = 0.0f;
            if (lane == 0) {
                for (uintptr_t p = a0; p < a1; p += kZeroChunk) {
                    const uintptr_t n = a1 - p < uintptr_t(kZeroChunk) ? a1 - p : uintptr_t(kZeroChunk);
                    bulk_store(reinterpret_cast<void*>(p), zero_sm, uint32_t(n));
                }
                bulk_commit_and_wait();
            }
        } else {
            for (uintptr_t p = b0 + 4 * lane; p < b1; p += 128) *reinterpret_cast<float*>(p) = 0.0f;
        }
    }
    const int scene = A.scene_of_world[w];
    const int64_t* meta = A.scene_meta + 8 * scene;
    const uint8_t* gbase = A.scene_blob + meta[0];
    const double ox = A.grid_offset[2 * w], oy = A.grid_offset[2 * w + 1];
    // scene-local geometry -> global (exactly mid + offset); per-world blobs
    // (geometry_global) were translated on the host
    const bool geo_global = A.d.geometry_global != 0;
    auto tx = [&](double v) { return geo_global ? v : v + ox; };
    auto ty = [&](double v) { return geo_global ? v : v + oy; };

    // ---- wait for the physics kernel (its writes are visible after this)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (kStep && world_ok[w] == 0) return;       // rejected actions: nothing mutates
    const int step_now = kStep ? world_step[w] : 0;
    for (int i = tid; i < M * int(sizeof(AgentRec) / 16); i += blockDim.x)
        reinterpret_cast<int4*>(ag)[i] = reinterpret_cast<const int4*>(rec + int64_t(w) * M)[i];
    __syncthreads();
    if (warp >= mc) return;

    const SceneView G = scene_view(const_cast<uint8_t*>(gbase), A.scene_blob + meta[5], int(meta[2]),
                                   int(meta[3]), int(meta[4]));
    const int m = m0 + warp;
    const int64_t am = int64_t(w) * M + m;
    const AgentRec& S = ag[m];
    float* row = rows + int64_t(warp) * D;
    const double px = S.x, py = S.y, c = S.c, s = S.s;
    const int road0 = A.d.ego_dim;
    const int veh0 = A.d.ego_dim + 5 * A.d.k_road;
    const bool rewards_needed = kStep && S.alive;
    int32_t* ix_m = A.index_out ? A.index_out + (int64_t(slot) * WM + am) * A.index_stride : nullptr;
    int16_t* px_m = A.prefix_out ? A.prefix_out + (int64_t(slot) * WM + am) * 2 : nullptr;

    // (1) neighbours: lane j <-> agent j (16 lanes), stable distance rank,
    //     swept TTC, neighbour row, hull contact
    double ttc_min;
    bool touch;
    {
        const int j = lane;
        double key = INFINITY, ndx = 0.0, ndy = 0.0;
        if (j < M) {
            const AgentRec& N = ag[j];
            ndx = N.x - px;
            ndy = N.y - py;
            const double dist = dg::dsqrt(ndx * ndx + ndy * ndy);
            key = (N.alive && j != m) ? dist : INFINITY;
        }
        int rank = 0;
        for (int t = 0; t < M; ++t) {
            const double kt = __shfl_sync(kFull, key, t);
            rank += (kt < key) || (kt == key && t < j);
        }
        const bool nvalid = j < M && finite(key) && rank < A.take_veh;
        if (ix_m || px_m) {
            if (ix_m && nvalid) ix_m[3 + rank] = j;
            const int nv = __popc(__ballot_sync(kFull, nvalid));
            if (ix_m && lane == 0) ix_m[2] = nv;
            if (px_m && lane == 0) px_m[1] = int16_t(7 * nv);
        }
        double ttc = k.ttc_max;
        if (nvalid) {
            const AgentRec& N = ag[j];
            ttc = swept_ttc(ndx, ndy, N.vwx - S.vwx, N.vwy - S.vwy, c, s, S.d, N.c, N.s, N.d, S.r + N.r,
                            k.ttc_max);
            const double wrap = wrap_angle(N.yaw - S.yaw);
            float* o = row + veh0 + 7 * rank;
            o[0] = __double2float_rn(dg::ddiv(c * ndx + s * ndy, k.bbox_half));
            o[1] = __double2float_rn(dg::ddiv(-s * ndx + c * ndy, k.bbox_half));
            o[2] = N.f_len;
            o[3] = N.f_wid;
            o[4] = __double2float_rn(dg::ddiv(wrap, 3.141592653589793));
            o[5] = N.f_spd;
            o[6] = __double2float_rn(dg::ddiv(ttc, k.ttc_max));
        }
        ttc_min = warp_min(ttc);
        bool t_ = false;
        if (kStep && j < M && j != m && S.alive && ag[j].alive &&
            key <= S.r + ag[j].r + S.d + ag[j].d + 1e-4) {
            const AgentRec& N = ag[j];
            const double rs = S.r + N.r;
            const double rs2 = rs * rs;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const double ex = S.hx[a] - N.hx[b], ey = S.hy[a] - N.hy[b];
                    t_ |= ex * ex + ey * ey < rs2;
                }
        }
        touch = __any_sync(kFull, t_);
        if (kStep && A.drac_max) {
            double dr = 0.0;
            if (j < M && j != m && S.alive && ag[j].alive) {
                const AgentRec& N = ag[j];
                dr = pair_drac(ndx, ndy, N.vwx - S.vwx, N.vwy - S.vwy, S.hx, S.hy, N.hx, N.hy, S.r + N.r);
            }
            dr = warp_max_nn(dr);
            if (lane == 0) {
                const double prev = A.drac_max[am];
                A.drac_max[am] = dr > prev ? dr : prev;
            }
        }
    }

    // (2) road context + edge boxes over the cell's superset list
    const double r2 = S.r * S.r;
    bool edge_hit = false;
    uint16_t* cand = cand_sm + warp * A.take_road;
    int count = 0;
    auto visit = [&](int q, bool in, bool edge_q) {
        bool hit = false;
        if (in) {
            const double2 m2 = __ldg(G.mid + q);
            const double mx = tx(m2.x), my = ty(m2.y);
            const double dx = mx - px, dy = my - py;
            const double d2 = dx * dx + dy * dy;
            hit = d2 <= k.road_radius_sq;
            if (rewards_needed && edge_q) {
                const double hl = __ldg(G.hl + q), hw = __ldg(G.hw + q);
                const double reach = S.r + S.d + hl + hw + 1e-6;
                if (d2 <= reach * reach) {
                    const double2 u2 = __ldg(G.dir + q);
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const double qx = S.hx[i] - mx, qy = S.hy[i] - my;
                        const double along = qx * u2.x + qy * u2.y;
                        const double lat = u2.x * qy - u2.y * qx;
                        const double du = along - sel_clip(along, -hl, hl);
                        const double dv = lat - sel_clip(lat, -hw, hw);
                        edge_hit |= du * du + dv * dv < r2;
                    }
                }
            }
        }
        const unsigned bal = __ballot_sync(kFull, hit);
        if (hit) {
            const int slot = count + __popc(bal & ((1u << lane) - 1u));
            if (slot < A.take_road) cand[slot] = uint16_t(q);
        }
        count += __popc(bal);
    };
    const bool use_grid = (G.flags & kFlagGrid) != 0;
    int cell_id = -1;
    if (G.flags) {
        const double inv = 1.0 / G.cell;
        const double fx = floor((px - ox - G.gx0) * inv), fy = floor((py - oy - G.gy0) * inv);
        if (fx >= 0.0 && fy >= 0.0 && fx < double(G.nx) && fy < double(G.ny)) cell_id = int(fy) * G.nx + int(fx);
    }
    if (use_grid) {
        if (cell_id >= 0) {
            const int lo = __ldg(G.road_start + cell_id), hi = __ldg(G.road_start + cell_id + 1);
            for (int b0 = lo; b0 < hi; b0 += 32) {
                const int i = b0 + lane;
                const int e = i < hi ? int(__ldg(G.road_list + i)) : 0;
                const int q = e & 0x7fff;
                const bool edge_q = (e >> 15) != 0;
                visit(q, i < hi, edge_q);
            }
        }
    } else {
        for (int p0 = 0; p0 < G.P; p0 += 32) visit(p0 + lane, p0 + lane < G.P, false);
    }
    const int ncand = count < A.take_road ? count : A.take_road;
    __syncwarp();
    if (ix_m && lane == 0) ix_m[1] = ncand;
    if (px_m && lane == 0) px_m[0] = int16_t(5 * ncand);
    for (int slot = lane; slot < ncand; slot += 32) {
        const int q = cand[slot];
        if (ix_m) ix_m[3 + A.take_veh + slot] = q;
        const double2 m2 = __ldg(G.mid + q), u2 = __ldg(G.dir + q);
        const double dx = (tx(m2.x)) - px, dy = (ty(m2.y)) - py;
        float* o = row + road0 + 5 * slot;
        o[0] = __double2float_rn(dg::ddiv(c * dx + s * dy, k.road_radius));
        o[1] = __double2float_rn(dg::ddiv(-s * dx + c * dy, k.road_radius));
        o[2] = __ldg(G.type_feat + q);
        o[3] = __double2float_rn(c * u2.x + s * u2.y);
        o[4] = __double2float_rn(-s * u2.x + c * u2.y);
    }

    // (3) the ego block (one lane)
    const double gx = A.goal_xy[2 * am], gy = A.goal_xy[2 * am + 1];
    if (lane == 0) write_ego(row, k, A, w, am, px, py, c, s, S.vx, S.vy, gx, gy);

    if constexpr (!kStep) {
        if (lane == 0 && A.ttc_min_out) A.ttc_min_out[am] = ttc_min;
        return;
    }

    // (4) rewards: first edge ahead, nearest lane (alive agents only)
    double gap = INFINITY, best = INFINITY;
    int best_k = 0x7fffffff;
    if (rewards_needed) {
#pragma unroll 2
        for (int kk = lane; kk < G.KE; kk += 32) {
            const double2 m2 = __ldg(G.edge_mid + kk);
            const double ex = (tx(m2.x)) - px, ey = (ty(m2.y)) - py;
            const double xb = c * ex + s * ey;
            if (xb > 0.0 && xb <= k.edge_range && xb < gap) gap = xb;
            if (!use_grid) {
                const int q = __ldg(G.edge + kk);
                const double2 u2 = __ldg(G.dir + q);
                const double hl = __ldg(G.hl + q), hw = __ldg(G.hw + q);
                const double reach = S.r + S.d + hl + hw + 1e-6;
                if (ex * ex + ey * ey <= reach * reach) {
                    const double mx = tx(m2.x), my = ty(m2.y);
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const double qx = S.hx[i] - mx, qy = S.hy[i] - my;
                        const double along = qx * u2.x + qy * u2.y;
                        const double lat = u2.x * qy - u2.y * qx;
                        const double du = along - sel_clip(along, -hl, hl);
                        const double dv = lat - sel_clip(lat, -hw, hw);
                        edge_hit |= du * du + dv * dv < r2;
                    }
                }
            }
        }
        gap = warp_min(gap);
        auto lane_test = [&](int kk) {
            const double4 l4 = ldg4(G.lane_seg + kk);
            const double ex = px - (tx(l4.x)), ey = py - (ty(l4.y));
            const double along = ex * l4.z + ey * l4.w;
            const double lat = l4.z * ey - l4.w * ex;
            const double t = fabs(along) - __ldg(G.lane_hl + kk);
            const double over = t > 0.0 ? t : 0.0;
            const double d2 = over * over + lat * lat;
            if (d2 < best) { best = d2; best_k = kk; }
        };
        const int lcell = (G.flags & kFlagLanes) ? cell_id : -1;
        if (lcell >= 0) {
            const int b0 = __ldg(G.lane_start + lcell), b1 = __ldg(G.lane_start + lcell + 1);
            for (int i = b0 + lane; i < b1; i += 32) lane_test(__ldg(G.lane_list + i));
        } else {
            for (int kk = lane; kk < G.KL; kk += 32) lane_test(kk);
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(kFull, best, o);
            const int ok = __shfl_xor_sync(kFull, best_k, o);
            if (ob < best || (ob == best && ok < best_k)) { best = ob; best_k = ok; }
        }
    }
    edge_hit = __any_sync(kFull, edge_hit);
    if (ix_m && lane == 0) ix_m[0] = rewards_needed && best < INFINITY ? best_k : -1;

    // (5) the agent's reward / event / termination tail
    if (lane == 0) {
        double st[DG_NUM_STATE];
#pragma unroll
        for (int f = 0; f < DG_NUM_STATE; ++f) st[f] = A.state[int64_t(f) * WM + am];
        FinIn F;
        F.st = st;
        F.c = S.c;
        F.s = S.s;
        F.px0 = prev[am].x; F.py0 = prev[am].y;
        F.gx = gx; F.gy = gy;
        F.sx = A.start_xy[2 * am]; F.sy = A.start_xy[2 * am + 1];
        F.lane_d2 = best;
        F.lane_lat = 0.0; F.lane_tx = 0.0; F.lane_ty = 0.0;
        if (best < INFINITY) {
            const double4 l4 = ldg4(G.lane_seg + best_k);
            const double ex = px - (tx(l4.x)), ey = py - (ty(l4.y));
            F.lane_tx = l4.z;
            F.lane_ty = l4.w;
            F.lane_lat = l4.z * ey - l4.w * ex;
        }
        F.ttc_min = ttc_min; F.gap = gap;
        F.edge_hit = edge_hit; F.touch = touch;
        F.alive = S.alive; F.valid = A.valid[am]; F.reason = A.reason[am]; F.seen = A.event_seen[am];
        F.spawn = A.spawn_step[am];
        F.start_yaw = A.start_yaw[am];
        F.store_global = true;
        F.st_out = nullptr;
        F.flags_out = nullptr;
        const unsigned bits = finalize_agent(A, tick_out(A, slot), w, m, F, step_now, ox, oy);
        count_events(A, w, bits, 1u, true, true);
    }
}

// ----------------------------------------------------------------- small kernels
__global__ void check_actions_kernel(const void* actions, int f64, int64_t n, int32_t* err) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double v = f64 ? reinterpret_cast<const double*>(actions)[i]
                             : double(reinterpret_cast<const float*>(actions)[i]);
        if (!isfinite(v)) atomicMin(err, int(i));
    }
}

// engine.py:599-619: masked slots get a fresh pose, zero velocity, cleared latches
__global__ void teleport_reset_kernel(KArgs A, const uint8_t* mask, const double* new_starts,
                                      const double* new_goals, const double* new_headings) {
    const int WM = A.d.W * A.d.M;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < WM; i += gridDim.x * blockDim.x) {
        const bool sel = (mask ? mask[i] != 0 : true) && A.valid[i];
        if (!sel) continue;
        double* sxy = A.start_xy;
        double* gxy = A.goal_xy;
        double* syaw = A.start_yaw;
        if (new_starts) { sxy[2 * i] = new_starts[2 * i]; sxy[2 * i + 1] = new_starts[2 * i + 1]; }
        if (new_goals) { gxy[2 * i] = new_goals[2 * i]; gxy[2 * i + 1] = new_goals[2 * i + 1]; }
        if (new_headings) syaw[i] = new_headings[i];
        for (int f = 0; f < DG_NUM_STATE; ++f) A.state[int64_t(f) * WM + i] = (f == SBF || f == SBR) ? 1.0 : 0.0;
        A.state[int64_t(SX) * WM + i] = sxy[2 * i];
        A.state[int64_t(SY) * WM + i] = sxy[2 * i + 1];
        A.state[int64_t(SYAW) * WM + i] = syaw[i];
        A.alive[i] = 1;
        A.reason[i] = 0;
        A.spawn_step[i] = A.step_count[i / A.d.M];
        A.event_seen[i] = 0;
    }
}

__global__ void set_step_kernel(int32_t* step_count, int W, int32_t value) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W; i += gridDim.x * blockDim.x) step_count[i] = value;
}

// policies.py:21-43 on the device, float64 like the numpy policy
// Standalone pairwise DRAC over logged states (metrics.py:33-62, 101-108):
// one CTA per world, 16 lanes per ego agent (lane j <-> other agent j), the
// world's records visited in order, the per-agent max kept in a register.
__global__ void __launch_bounds__(256) pairwise_drac_kernel(const double* x, const double* y, const double* yaw,
                                                            const double* vx, const double* vy,
                                                            const uint8_t* alive, const double* r_hull,
                                                            const double* d_hull, int steps, int W, int M,
                                                            double* out, int accumulate, int world_vel) {
    __shared__ double s_px[kMaxAgents], s_py[kMaxAgents], s_ux[kMaxAgents], s_uy[kMaxAgents];
    __shared__ double s_hx[kMaxAgents][3], s_hy[kMaxAgents][3];
    __shared__ int s_alive[kMaxAgents];
    const int w = blockIdx.x;
    const int i = threadIdx.x >> 4, j = threadIdx.x & 15;
    const int64_t WM = int64_t(W) * M;
    double best = 0.0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x < M) {
            const int m = threadIdx.x;
            const int64_t q = t * WM + int64_t(w) * M + m;
            const double px = x[q], py = y[q], th = yaw[q], bx = vx[q], by = vy[q];
            const double c = cos(th), sn = sin(th);                 // metrics.py:104
            s_px[m] = px;
            s_py[m] = py;
            s_ux[m] = world_vel ? bx : bx * c - by * sn;             // metrics.py:105-106
            s_uy[m] = world_vel ? by : bx * sn + by * c;
            const double d = d_hull[int64_t(w) * M + m];
            const double oc = d * c, os = d * sn;                    // metrics.py:46-49
            s_hx[m][0] = px + -1.0 * oc; s_hx[m][1] = px + 0.0 * oc; s_hx[m][2] = px + 1.0 * oc;
            s_hy[m][0] = py + -1.0 * os; s_hy[m][1] = py + 0.0 * os; s_hy[m][2] = py + 1.0 * os;
            s_alive[m] = alive[q];
        }
        __syncthreads();
        double dr = 0.0;
        if (i < M && j < M && i != j && s_alive[i] && s_alive[j]) {
            dr = pair_drac(s_px[j] - s_px[i], s_py[j] - s_py[i], s_ux[j] - s_ux[i], s_uy[j] - s_uy[i], s_hx[i],
                           s_hy[i], s_hx[j], s_hy[j], r_hull[int64_t(w) * M + i] + r_hull[int64_t(w) * M + j]);
        }
        dr = warp_max_nn(dr, 16);
        best = dr > best ? dr : best;
        __syncthreads();
    }
    if (i < M && j == 0) {
        double* p = out + int64_t(w) * M + i;
        if (accumulate) {
            const double prev = *p;
            best = best > prev ? best : prev;
        }
        *p = best;
    }
}

// Batched system-identification rollouts (sysid.py:201-228): thread (b, m) rolls
// maneuver m for candidate parameter vector b -- the step kernel's 120 Hz
// substep with that candidate's constant block -- and records the 7 channels
// after every second substep (60 Hz).  out + out_offset[m] holds [7][2 T_m][B].
__global__ void __launch_bounds__(64) sysid_rollout_kernel(const DgConsts* consts, const double* mu,
                                                           const int32_t* tick_start, const double* actions,
                                                           const uint8_t* surface, const int64_t* out_offset,
                                                           int B, double* out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = blockIdx.y;
    if (b >= B) return;
    const DgConsts k = consts[b];
    const Rcp rc = make_rcp(k);           // this candidate's constants
    double x[DG_NUM_STATE];
#pragma unroll
    for (int f = 0; f < DG_NUM_STATE; ++f) x[f] = 0.0;
    x[SBF] = 1.0;
    x[SBR] = 1.0;
    const int t0 = tick_start[m], t1 = tick_start[m + 1];
    const int64_t T60 = 2 * int64_t(t1 - t0);
    double* o = out + out_offset[m];
    int64_t rec = 0;
    for (int t = t0; t < t1; ++t) {
        Act a;
        a.thr = actions[3 * t];
        a.steer = actions[3 * t + 1];
        a.brk = actions[3 * t + 2];
        const double cap = mu[3 * b + surface[t]] * k.f_z;
        for (int sub = 0; sub < 4; ++sub) {
            substep_dynamic(x, a, cap, k, rc);
            if (sub & 1) {
                double* r = o + rec * B + b;
                r[0 * T60 * B] = x[SX];
                r[1 * T60 * B] = x[SY];
                r[2 * T60 * B] = x[SYAW];
                r[3 * T60 * B] = sqrt(x[SVX] * x[SVX] + x[SVY] * x[SVY]);
                r[4 * T60 * B] = x[SOM];
                r[5 * T60 * B] = 0.5 * (x[SWF] + x[SWR]);
                r[6 * T60 * B] = x[SANG];
                ++rec;
            }
        }
    }
}

__global__ void lane_follower_kernel(const float* obs, double* actions, int64_t n, int D, double gain,
                                     double throttle, double bbox_half) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float* o = obs + i * D;
        const double sin_e = double(o[2]), cos_e = double(o[3]);
        const double dist = double(o[4]) * bbox_half;
        double steer = np_clip(gain * sin_e, -1.0, 1.0);
        if (cos_e < 0.0) steer = sin_e >= 0.0 ? 1.0 : -1.0;
        actions[3 * i] = dist > 5.0 ? throttle : throttle * 0.5;
        actions[3 * i + 1] = steer;
        actions[3 * i + 2] = 0.0;
    }
}

}  // namespace


// ----------------------------------------------------------------- host delivery of observations
// The numpy step path (engine.py:297-335 returns host arrays) moves the
// observation to a mapped pinned host slab without carrying its zero tails
// over PCIe: every row is [ego | road 5*k_road | vehicles 7*k_veh] and the
// kernel writes road / vehicle slots prefix-compacted over a zero background,
// so per block only the prefix up to the last non-zero float (bitwise: -0.0
// and NaN count as non-zero) has to cross the link.  The slab keeps, per row,
// the prefix lengths it currently holds (prev, device memory); a row whose
// new prefix is shorter gets zeros over the difference, so the slab equals the
// device rows bit for bit after every call.  One warp per row; stores to the
// host are 32 consecutive floats per instruction.
__device__ __forceinline__ int last_nonzero_prefix(const float* p, int n, int lane) {
    int last = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const bool nz = i < n && __float_as_uint(__ldg(p + i)) != 0u;
        const unsigned b = __ballot_sync(kFull, nz);
        if (b) last = i0 + 32 - __clz(b);
    }
    return last;
}

// src and dst share their alignment modulo 16 bytes (row offsets are equal and
// both bases are 16-byte aligned): scalar head, 16-byte body, scalar tail.
__device__ __forceinline__ void copy_to_host(const float* src, float* dst, int n, int lane) {
    if (n <= 0) return;
    int head = int((16u - unsigned(reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u) >> 2;
    head = head < n ? head : n;
    if (lane < head) dst[lane] = __ldg(src + lane);
    const float4* s4 = reinterpret_cast<const float4*>(src + head);
    float4* d4 = reinterpret_cast<float4*>(dst + head);
    const int n4 = (n - head) >> 2;
    for (int i = lane; i < n4; i += 32) d4[i] = __ldg(s4 + i);
    const int done = head + 4 * n4;
    if (lane < n - done) dst[done + lane] = __ldg(src + done + lane);
}

__device__ __forceinline__ void zero_host(float* dst, int n, int lane) { zero_span(dst, n, lane, 32); }

__global__ void __launch_bounds__(256) obs_to_host_kernel(const float* obs, const int16_t* prefix, float* host,
                                                          int32_t* prev, int64_t rows, int D, int ego, int road_n,
                                                          int veh_n, unsigned long long* bytes) {
    const int lane = threadIdx.x & 31;
    const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float* src = obs + r * D;
    float* dst = host + r * D;
    const int lr = prefix ? min(int(prefix[2 * r]), road_n) : last_nonzero_prefix(src + ego, road_n, lane);
    const int lv = prefix ? min(int(prefix[2 * r + 1]), veh_n) : last_nonzero_prefix(src + ego + road_n, veh_n, lane);
    const int pr = prev[2 * r], pv = prev[2 * r + 1];
    copy_to_host(src, dst, ego + lr, lane);
    if (pr > lr) zero_host(dst + ego + lr, pr - lr, lane);
    copy_to_host(src + ego + road_n, dst + ego + road_n, lv, lane);
    if (pv > lv) zero_host(dst + ego + road_n + lv, pv - lv, lane);
    if (lane == 0) {
        prev[2 * r] = lr;
        prev[2 * r + 1] = lv;
        if (bytes) {
            const int n = ego + lr + (pr > lr ? pr - lr : 0) + lv + (pv > lv ? pv - lv : 0);
            atomicAdd(bytes, 4ull * unsigned(n));
        }
    }
}

// =========================================================================== C ABI

struct dg_engine {
    DgEngineDesc desc;
    KArgs base;
    size_t smem_bytes;
    int launches;
    int warps_per_world;   // fused: CTA = warps_per_world warps; split: agents (warps) per CTA
    int min_blocks;        // register budget: resident CTAs per SM the variant is built for
    int mode;              // 0 = fused world kernel, 1 = split physics + per-agent kernels (PDL),
                           // 2 = fused with a physics warp running one tick ahead (kSpec)
    size_t smem_split;     // dynamic smem of the per-agent kernel
    // dg_to_host: the packed per-tick outputs go down on a side stream while the
    // obs rows are written into the slab (the SM stores leave PCIe headroom)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_aux = nullptr;
    ~dg_engine() {
        if (ev_ready) cudaEventDestroy(ev_ready);
        if (ev_aux) cudaEventDestroy(ev_aux);
        if (side) cudaStreamDestroy(side);
    }
};

// the shapes the engine picks by default also come with the phase counters
#define DG_PHASE_VARIANTS(X) X(256, 2, true, false) X(256, 2, false, false) X(128, 4, false, false)

#define DG_VARIANTS(X)                                                                 \
    X(512, 1, false, false) X(512, 2, false, false) X(256, 2, false, false) X(256, 3, false, false) \
    X(256, 4, false, false) X(128, 4, false, false) X(128, 6, false, false) X(128, 8, false, false) \
    X(256, 2, true, false) X(256, 2, false, true) X(128, 4, false, true) X(256, 2, true, true)

// Kernel variants: (threads per CTA, min resident CTAs per SM) bounds trade
// registers for occupancy; dg_tune picks one.  The kSpec variant is up to 7
// scan warps plus the physics warp (256 threads: 128 registers at 2 CTAs/SM).
static int variant_threads(int nw, bool spec) { return spec ? 256 : (nw > 8 ? 512 : (nw > 4 ? 256 : 128)); }

template <bool kStep>
static cudaError_t launch_world_step(const dg_engine* e, const KArgs& A, cudaStream_t st) {
    const int nw = e->warps_per_world;
    const bool spec = e->mode == 2;
    const bool geo = A.d.geometry_global != 0;
    const int threads = variant_threads(nw, spec);
    const dim3 grid(A.d.W);
    if (A.phase_cycles) {
#define DG_LAUNCH_PH(T, B, S, G)                                                         \
        if (threads == T && e->min_blocks == B && spec == S && geo == G) {               \
            world_step_kernel<kStep, T, B, S, G, true><<<grid, 32 * (nw + (S ? 1 : 0)), e->smem_bytes, st>>>(A); \
            return cudaGetLastError();                                                   \
        }
        DG_PHASE_VARIANTS(DG_LAUNCH_PH)
#undef DG_LAUNCH_PH
    }
#define DG_LAUNCH(T, B, S, G)                                                            \
    if (threads == T && e->min_blocks == B && spec == S && geo == G) {                   \
        world_step_kernel<kStep, T, B, S, G><<<grid, 32 * (nw + (S ? 1 : 0)), e->smem_bytes, st>>>(A); \
        return cudaGetLastError();                                                       \
    }
    DG_VARIANTS(DG_LAUNCH)
#undef DG_LAUNCH
    return cudaErrorInvalidConfiguration;
}

// Raise a kernel's dynamic shared-memory limit to the device ceiling (opt-in
// per-block maximum minus the kernel's static shared memory).
template <typename K>
static cudaError_t raise_smem_limit(K kernel) {
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kernel);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - int(fa.sharedSizeBytes));
    return e;
}

template <bool kStep>
static cudaError_t set_smem_attr(size_t) {
    cudaError_t e = cudaSuccess;
#define DG_ATTR(T, B, S, G)                                                              \
    if (e == cudaSuccess) e = raise_smem_limit(world_step_kernel<kStep, T, B, S, G>);
    DG_VARIANTS(DG_ATTR)
#undef DG_ATTR
#define DG_ATTR(T, B, S, G)                                                              \
    if (e == cudaSuccess) e = raise_smem_limit(world_step_kernel<kStep, T, B, S, G, true>);
    DG_PHASE_VARIANTS(DG_ATTR)
#undef DG_ATTR
    return e;
}

static bool has_variant(int threads, int blocks, bool spec, bool geo) {
#define DG_HAS(T, B, S, G) if (threads == T && blocks == B && spec == S && geo == G) return true;
    DG_VARIANTS(DG_HAS)
#undef DG_HAS
    return false;
}

// split mode: per-agent kernel variants (threads = 32 * agents per CTA)
#define DG_SPLIT_VARIANTS(X) X(64, 8) X(64, 12) X(64, 16) X(128, 4) X(128, 6) X(128, 8) X(256, 2) X(256, 4)

static bool has_split_variant(int threads, int blocks) {
#define DG_HAS(T, B) if (threads == T && blocks == B) return true;
    DG_SPLIT_VARIANTS(DG_HAS)
#undef DG_HAS
    return false;
}

template <bool kStep>
static cudaError_t set_split_smem_attr(size_t) {
    cudaError_t e = cudaSuccess;
#define DG_ATTR(T, B)                                                                    \
    if (e == cudaSuccess) e = raise_smem_limit(agent_obs_kernel<kStep, T, B>);
    DG_SPLIT_VARIANTS(DG_ATTR)
#undef DG_ATTR
    return e;
}

template <bool kStep>
static cudaError_t launch_split(const dg_engine* e, const KArgs& A, cudaStream_t st) {
    world_physics_kernel<kStep><<<A.d.W, 32, 0, st>>>(A);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    const int apc = e->warps_per_world;
    const int threads = 32 * apc;
    const int groups = (A.d.M + apc - 1) / apc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(A.d.W * groups);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = e->smem_split;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define DG_LAUNCH(T, B)                                                                  \
    if (threads == T && e->min_blocks == B) return cudaLaunchKernelEx(&cfg, agent_obs_kernel<kStep, T, B>, A);
    DG_SPLIT_VARIANTS(DG_LAUNCH)
#undef DG_LAUNCH
    return cudaErrorInvalidConfiguration;
}

template <bool kStep>
static cudaError_t launch_step_any(const dg_engine* e, const KArgs& A, cudaStream_t st) {
    return e->mode == 1 ? launch_split<kStep>(e, A, st) : launch_world_step<kStep>(e, A, st);   // 0, 2: fused
}

// engine creation: the refined reciprocals of the constant divisors (Rcp)
__device__ Rcp g_rcp_out;
__global__ void rcp_kernel(const DgConsts k) { g_rcp_out = make_rcp(k); }

static thread_local char g_err[512] = "";

static int fail(int code, const char* msg) {
    std::snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

static int cuda_fail(cudaError_t e, const char* where) {
    std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return DG_ECUDA;
}

// error reporting for the library's other translation units (dg_worlds.cu)
int dg_internal_fail(int code, const char* msg) { return fail(code, msg); }
int dg_internal_cuda_fail(cudaError_t e, const char* where) { return cuda_fail(e, where); }

static size_t split_smem_bytes(int take_road, int apc) {
    size_t b = sizeof(AgentRec) * kMaxAgents;
    b += sizeof(uint16_t) * size_t(apc) * size_t(take_road > 0 ? take_road : 1);
    return size_t(align16(int64_t(b))) + kZeroChunk;
}

static size_t step_smem_bytes(const DgDims& d, int take_road) {
    size_t b = d.geometry_global ? 0 : size_t(align16(d.max_scene_bytes));   // global: read in place
    b += sizeof(AgentSm) * 3 * kMaxAgents;                                  // three agent tables
    b += sizeof(ScanSm) * 2 * kMaxAgents + sizeof(TailRes) * kMaxAgents;   // scan results x2, tail decisions
    b += 16;  // mbarrier
    b += sizeof(uint16_t) * kMaxAgents * size_t(take_road > 0 ? take_road : 1);
    b = size_t(align16(int64_t(b))) + kZeroChunk;
    b += sizeof(int16_t) * kPfxSlots * kMaxAgents * 2;   // resident-ring prefix cache
    return b;
}

extern "C" {

int dg_abi_version(void) { return DG_ABI_VERSION; }
const char* dg_last_error(void) { return g_err; }

int dg_create(const DgEngineDesc* desc, dg_engine** out) {
    if (!desc || !out) return fail(DG_EINVAL, "dg_create: null argument");
    const DgDims& d = desc->dims;
    if (d.W < 1 || d.M < 1 || d.M > kMaxAgents) return fail(DG_EINVAL, "dg_create: need W >= 1 and 1 <= M <= 16");
    if (d.obs_dim != d.ego_dim + 5 * d.k_road + 7 * d.k_vehicles)
        return fail(DG_EINVAL, "dg_create: obs_dim != ego_dim + 5*k_road + 7*k_vehicles");
    if (d.ego_dim != 7 + (d.include_weather ? 4 : 0)) return fail(DG_EINVAL, "dg_create: bad ego_dim");
    if (d.max_segments > 65535) return fail(DG_ENOSUPPORT, "dg_create: more than 65535 segments in a scene");
    if (d.max_scene_bytes % 16) return fail(DG_EINVAL, "dg_create: scene blobs must be 16-byte multiples");
    const void* req[] = {desc->scene_blob, desc->scene_meta, desc->scene_of_world, desc->grid_offset,
                         desc->mu_eff, desc->weather, desc->valid, desc->length, desc->width,
                         desc->r_hull, desc->d_hull, desc->state, desc->alive, desc->reason,
                         desc->event_seen, desc->spawn_step, desc->step_count, desc->start_xy,
                         desc->goal_xy, desc->start_yaw, desc->error_word};
    for (const void* p : req)
        if (!p) return fail(DG_EINVAL, "dg_create: null device pointer in engine description");

    dg_engine* e = new (std::nothrow) dg_engine();
    if (!e) return fail(DG_ECUDA, "dg_create: out of host memory");
    e->desc = *desc;
    KArgs& A = e->base;
    std::memset(&A, 0, sizeof(A));
    A.d = d;
    A.k = desc->k;
    {
        // the constant divisors' refined reciprocals, as the GPU computes them
        static std::mutex rcp_mu;
        std::lock_guard<std::mutex> lock(rcp_mu);
        rcp_kernel<<<1, 1>>>(desc->k);
        cudaError_t rerr = cudaGetLastError();
        if (rerr == cudaSuccess) rerr = cudaMemcpyFromSymbol(&A.rc, g_rcp_out, sizeof(Rcp));
        if (rerr != cudaSuccess) {
            delete e;
            return cuda_fail(rerr, "dg_create: reciprocal constants");
        }
    }
    A.scene_blob = desc->scene_blob;
    A.scene_meta = desc->scene_meta;
    A.scene_of_world = desc->scene_of_world;
    A.grid_offset = desc->grid_offset;
    A.mu_eff = desc->mu_eff;
    A.weather = desc->weather;
    A.valid = desc->valid;
    A.length = desc->length;
    A.width = desc->width;
    A.r_hull = desc->r_hull;
    A.d_hull = desc->d_hull;
    A.state = desc->state;
    A.alive = desc->alive;
    A.reason = desc->reason;
    A.event_seen = desc->event_seen;
    A.spawn_step = desc->spawn_step;
    A.step_count = desc->step_count;
    A.start_xy = desc->start_xy;
    A.goal_xy = desc->goal_xy;
    A.start_yaw = desc->start_yaw;
    A.error_word = desc->error_word;
    A.scratch = desc->scratch;
    A.take_road = d.k_road < d.max_segments ? d.k_road : d.max_segments;
    A.take_veh = d.k_vehicles < d.M ? d.k_vehicles : d.M;
    A.index_stride = 3 + A.take_veh + A.take_road;
    e->smem_bytes = step_smem_bytes(d, A.take_road);
    // headroom for the kernels' static / reserved shared memory
    if (!d.geometry_global && e->smem_bytes > 227 * 1024 - 4096) {
        delete e;
        return fail(DG_ENOSUPPORT, "dg_create: scene geometry does not fit in shared memory");
    }
    e->smem_split = split_smem_bytes(A.take_road, 8);
    // The attribute belongs to the kernel, not the engine: always the device
    // ceiling, so engines with smaller blobs never shrink another engine's limit
    // (each launch passes its own dynamic size; occupancy follows that size).
    cudaError_t err = set_smem_attr<true>(0);
    if (err == cudaSuccess) err = set_smem_attr<false>(0);
    if (err == cudaSuccess) err = set_split_smem_attr<true>(0);
    if (err == cudaSuccess) err = set_split_smem_attr<false>(0);
    if (err != cudaSuccess) {
        delete e;
        return cuda_fail(err, "dg_create: cudaFuncSetAttribute");
    }
    e->launches = 0;
    e->warps_per_world = d.M;
    e->min_blocks = 1;
    e->mode = 0;
    if (d.geometry_global) {
        // per-world blobs stay in global memory, read in place: by the split
        // kernels when the scratch buffer is there (measured 2x faster than the
        // fused kernel's kGeoGlobal variants on the dense 6,000-segment scene:
        // a warp per agent beats a 16-lane group on 350-row road blocks), else
        // by the fused kernel (dg_tune picks either later)
        e->mode = A.scratch ? 1 : 0;
        e->warps_per_world = 4 < d.M ? 4 : d.M;
        e->min_blocks = 4;
    }
    *out = e;
    return DG_OK;
}

int dg_destroy(dg_engine* eng) {
    delete eng;
    return DG_OK;
}

int dg_step(dg_engine* eng, const DgStepIO* io, void* stream) {
    if (!eng || !io) return fail(DG_EINVAL, "dg_step: null argument");
    if (!io->actions || !io->obs || !io->rewards || !io->dones || !io->events)
        return fail(DG_EINVAL, "dg_step: actions, obs, rewards, dones and events are required");
    KArgs A = eng->base;
    A.actions = io->actions;
    A.actions_f64 = io->actions_f64;
    A.autoreset = io->autoreset;
    A.obs = io->obs;
    A.rewards = io->rewards;
    A.dones = io->dones;
    A.events = io->events;
    A.reason_out = io->reason_out;
    A.alive_out = io->alive_out;
    A.alive_pre_out = io->alive_pre_out;
    A.ttc_min_out = io->ttc_min_out;
    A.terms_out = io->terms_out;
    A.snapshot_out = io->snapshot_out;
    A.next_actions = io->next_actions;
    A.event_counts = io->event_counts;
    A.pol_gain = io->policy_gain;
    A.pol_throttle = io->policy_throttle;
    A.drac_max = io->drac_max;
    A.metric_seen = io->metric_seen;
    A.index_out = io->index_out;
    A.prefix_out = io->prefix_out;
    A.obs_resident = io->obs_resident && io->prefix_out && eng->mode != 1;
    A.phase_cycles = reinterpret_cast<unsigned long long*>(io->phase_cycles);
    A.ticks = io->ticks > 0 ? io->ticks : 1;
    A.ring_slots = io->ring_slots > 0 ? io->ring_slots : A.ticks;
    A.ring_start = io->ring_start;
    if (A.ring_start < 0 || A.ring_start >= A.ring_slots)
        return fail(DG_EINVAL, "dg_step: ring_start must lie in [0, ring_slots)");
    if (A.ticks > 1 && eng->mode == 1)
        return fail(DG_ENOSUPPORT, "dg_step: ticks > 1 needs the fused launch mode");
    eng->launches = 1;
    const cudaError_t err = launch_step_any<true>(eng, A, static_cast<cudaStream_t>(stream));
    eng->launches = eng->mode == 1 ? 2 : 1;
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_step");
}

int dg_observe(dg_engine* eng, float* obs, double* ttc_min_out, double* next_actions, double policy_gain,
               double policy_throttle, void* stream) {
    if (!eng || !obs) return fail(DG_EINVAL, "dg_observe: null argument");
    KArgs A = eng->base;
    A.obs = obs;
    A.ttc_min_out = ttc_min_out;
    A.next_actions = next_actions;
    A.pol_gain = policy_gain;
    A.pol_throttle = policy_throttle;
    A.ticks = 1;
    A.ring_slots = 1;
    A.ring_start = 0;
    eng->launches = 1;
    const cudaError_t err = launch_step_any<false>(eng, A, static_cast<cudaStream_t>(stream));
    eng->launches = eng->mode == 1 ? 2 : 1;
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_observe");
}

int dg_reset(dg_engine* eng, const uint8_t* mask, const double* new_starts, const double* new_goals,
             const double* new_headings, void* stream) {
    if (!eng) return fail(DG_EINVAL, "dg_reset: null engine");
    const int WM = eng->base.d.W * eng->base.d.M;
    const int threads = 256, blocks = (WM + threads - 1) / threads;
    teleport_reset_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
        eng->base, mask, new_starts, new_goals, new_headings);
    eng->launches = 1;
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_reset");
}

int dg_set_step_count(dg_engine* eng, int32_t value, void* stream) {
    if (!eng) return fail(DG_EINVAL, "dg_set_step_count: null engine");
    const int W = eng->base.d.W;
    set_step_kernel<<<(W + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(eng->base.step_count, W, value);
    eng->launches = 1;
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_set_step_count");
}

int dg_check_actions(dg_engine* eng, const void* actions, int32_t actions_f64, void* stream) {
    if (!eng || !actions) return fail(DG_EINVAL, "dg_check_actions: null argument");
    const int64_t n = int64_t(eng->base.d.W) * eng->base.d.M * 3;
    const int threads = 256;
    const int blocks = int((n + threads - 1) / threads < 1184 ? (n + threads - 1) / threads : 1184);
    check_actions_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(actions, actions_f64, n,
                                                                                eng->base.error_word);
    eng->launches = 1;
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_check_actions");
}

int dg_read_error(dg_engine* eng, int32_t* flat_index, void* stream) {
    if (!eng || !flat_index) return fail(DG_EINVAL, "dg_read_error: null argument");
    int32_t host = DG_NO_ERROR;
    const int32_t clean = DG_NO_ERROR;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t err = cudaMemcpyAsync(&host, eng->base.error_word, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (err == cudaSuccess) err = cudaStreamSynchronize(s);
    if (err == cudaSuccess && host != DG_NO_ERROR)
        err = cudaMemcpyAsync(eng->base.error_word, &clean, sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) err = cudaStreamSynchronize(s);
    if (err != cudaSuccess) return cuda_fail(err, "dg_read_error");
    *flat_index = host == DG_NO_ERROR ? -1 : host;
    return DG_OK;
}

int dg_lane_follower(dg_engine* eng, const float* obs, double* actions, double steer_gain, double throttle,
                     void* stream) {
    if (!eng || !obs || !actions) return fail(DG_EINVAL, "dg_lane_follower: null argument");
    const int64_t n = int64_t(eng->base.d.W) * eng->base.d.M;
    const int threads = 128;
    const int blocks = int((n + threads - 1) / threads);
    lane_follower_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
        obs, actions, n, eng->base.d.obs_dim, steer_gain, throttle, eng->base.k.bbox_half);
    eng->launches = 1;
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_lane_follower");
}

int dg_pairwise_drac(const double* x, const double* y, const double* yaw, const double* v_x, const double* v_y,
                     const uint8_t* alive, const double* r_hull, const double* d_hull, int32_t steps, int32_t W,
                     int32_t M, double* out, int32_t accumulate, int32_t world_velocity, void* stream) {
    if (!x || !y || !yaw || !v_x || !v_y || !alive || !r_hull || !d_hull || !out)
        return fail(DG_EINVAL, "dg_pairwise_drac: null argument");
    if (W < 1 || M < 1 || M > kMaxAgents || steps < 0)
        return fail(DG_EINVAL, "dg_pairwise_drac: need W >= 1, 1 <= M <= 16, steps >= 0");
    pairwise_drac_kernel<<<W, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, y, yaw, v_x, v_y, alive, r_hull,
                                                                           d_hull, steps, W, M, out, accumulate,
                                                                           world_velocity);
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_pairwise_drac");
}

int dg_sysid_rollout(const void* consts, const double* mu, const int32_t* tick_start, const double* actions,
                     const uint8_t* surface, const int64_t* out_offset, int32_t B, int32_t n_maneuvers,
                     double* out, void* stream) {
    if (!consts || !mu || !tick_start || !actions || !surface || !out_offset || !out)
        return fail(DG_EINVAL, "dg_sysid_rollout: null argument");
    if (B < 1 || n_maneuvers < 1 || n_maneuvers > 65535)
        return fail(DG_EINVAL, "dg_sysid_rollout: need B >= 1 and 1 <= n_maneuvers <= 65535");
    const dim3 grid((B + 63) / 64, n_maneuvers);
    sysid_rollout_kernel<<<grid, 64, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const DgConsts*>(consts), mu, tick_start, actions, surface, out_offset, B, out);
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? DG_OK : cuda_fail(err, "dg_sysid_rollout");
}

int dg_get_state(dg_engine* eng, double* dst, void* stream) {
    if (!eng || !dst) return fail(DG_EINVAL, "dg_get_state: null argument");
    const size_t n = size_t(DG_NUM_STATE) * eng->base.d.W * eng->base.d.M * sizeof(double);
    const cudaError_t e = cudaMemcpyAsync(dst, eng->base.state, n, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DG_OK : cuda_fail(e, "dg_get_state");
}

int dg_set_state(dg_engine* eng, const double* src, void* stream) {
    if (!eng || !src) return fail(DG_EINVAL, "dg_set_state: null argument");
    const size_t n = size_t(DG_NUM_STATE) * eng->base.d.W * eng->base.d.M * sizeof(double);
    const cudaError_t e = cudaMemcpyAsync(eng->base.state, src, n, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? DG_OK : cuda_fail(e, "dg_set_state");
}


int dg_host_alloc(size_t bytes, void** host_ptr) {
    if (!host_ptr) return fail(DG_EINVAL, "dg_host_alloc: null output pointer");
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return cuda_fail(e, "dg_host_alloc");
    std::memset(p, 0, bytes);
    *host_ptr = p;
    return DG_OK;
}

int dg_host_free(void* host_ptr) {
    if (!host_ptr) return DG_OK;
    const cudaError_t e = cudaFreeHost(host_ptr);
    return e == cudaSuccess ? DG_OK : cuda_fail(e, "dg_host_free");
}

int dg_to_host(dg_engine* eng, const float* obs, const int16_t* prefix, float* host_obs, int32_t* prev_len,
               const void* aux, void* host_aux, size_t aux_bytes, unsigned long long* bytes, void* stream) {
    if (!eng || !obs || !host_obs || !prev_len) return fail(DG_EINVAL, "dg_to_host: null argument");
    if (aux_bytes && (!aux || !host_aux)) return fail(DG_EINVAL, "dg_to_host: null aux buffer");
    const DgDims& d = eng->base.d;
    void* dptr = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dptr, host_obs, 0);
    if (e != cudaSuccess) return cuda_fail(e, "dg_to_host: host slab is not mapped pinned memory");
    const int64_t rows = int64_t(d.W) * d.M;
    const int per_cta = 8;           // 1..16 rows per CTA measured the same (PCIe-bound)
    const int64_t grid = (rows + per_cta - 1) / per_cta;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (aux_bytes) {
        // fork: the aux DMA on the engine's side stream, concurrent with the row stores
        if (!eng->side) {
            e = cudaStreamCreateWithFlags(&eng->side, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&eng->ev_ready, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&eng->ev_aux, cudaEventDisableTiming);
            if (e != cudaSuccess) return cuda_fail(e, "dg_to_host: side stream");
        }
        e = cudaEventRecord(eng->ev_ready, st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(eng->side, eng->ev_ready, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(host_aux, aux, aux_bytes, cudaMemcpyDeviceToHost, eng->side);
        if (e == cudaSuccess) e = cudaEventRecord(eng->ev_aux, eng->side);
        if (e != cudaSuccess) return cuda_fail(e, "dg_to_host: aux copy");
    }
    if (grid > 0)
        obs_to_host_kernel<<<unsigned(grid), 32 * per_cta, 0, st>>>(
            obs, prefix, static_cast<float*>(dptr), prev_len, rows, d.obs_dim, d.ego_dim, 5 * d.k_road,
            7 * d.k_vehicles, bytes);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "dg_to_host");
    if (aux_bytes) {
        e = cudaStreamWaitEvent(st, eng->ev_aux, 0);     // join: the stream's sync covers both
        if (e != cudaSuccess) return cuda_fail(e, "dg_to_host: join");
    }
    return DG_OK;
}

// The numpy step path in one call (Engine._step_host; engine.py:334-406 behind
// env.py:48-65): the caller's float64 actions are checked for finiteness while
// they are copied into the pinned staging buffer (engine.py:291-294: a
// non-finite value returns DG_ENONFINITE with its flat index before anything is
// launched or mutated), then the H2D copy, the step and the host delivery are
// queued on one stream -- one host call instead of four.
int dg_step_host(dg_engine* eng, const DgStepIO* io, const double* host_actions, double* pinned_actions,
                 float* host_obs, int32_t* prev_len, const void* aux, void* host_aux, size_t aux_bytes,
                 unsigned long long* bytes, int64_t* bad_index, void* stream) {
    if (!eng || !io || !host_actions || !pinned_actions || !bad_index)
        return fail(DG_EINVAL, "dg_step_host: null argument");
    if (!io->actions_f64 || !io->actions) return fail(DG_EINVAL, "dg_step_host: io must carry float64 device actions");
    const DgDims& d = eng->base.d;
    const int64_t n = int64_t(d.W) * d.M * 3;
    *bad_index = -1;
    bool ok = true;
    for (int64_t i = 0; i < n; ++i) {
        const double a = host_actions[i];
        pinned_actions[i] = a;
        ok &= std::isfinite(a);
    }
    if (!ok) {
        for (int64_t i = 0; i < n; ++i)
            if (!std::isfinite(host_actions[i])) { *bad_index = i; break; }
        return fail(DG_ENONFINITE, "dg_step_host: non-finite action");
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the kernel reads the staged actions in place over PCIe (pinned host memory is
    // device-mapped under unified addressing): no copy launch ahead of the step; a
    // buffer without a device mapping goes through an H2D copy into io->actions
    DgStepIO sio = *io;
    void* mapped = nullptr;
    if (cudaHostGetDevicePointer(&mapped, pinned_actions, 0) == cudaSuccess && mapped) {
        sio.actions = mapped;
    } else {
        (void)cudaGetLastError();
        cudaError_t e = cudaMemcpyAsync(const_cast<void*>(io->actions), pinned_actions,
                                        size_t(n) * sizeof(double), cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "dg_step_host: action copy");
    }
    int rc = dg_step(eng, &sio, stream);
    if (rc != DG_OK || !host_obs) return rc;
    const int launches = eng->launches;
    rc = dg_to_host(eng, io->obs, io->prefix_out, host_obs, prev_len, aux, host_aux, aux_bytes, bytes, stream);
    eng->launches = launches + 1;
    return rc;
}

#ifndef DG_LF_PREFETCH
#define DG_LF_PREFETCH 16      // rows ahead: the slab rows arrive from the device, not in cache
#endif
// Host LaneFollower (policies.py:21-43) over float32 observation rows [rows][D]:
// float64 arithmetic as the numpy expression -- np.clip(gain * sin, -1, 1) as
// minimum(maximum(x, -1), 1), the goal-behind override, the distance-dependent
// throttle -- NaN and -0.0 included; one pass, each row's ego features read once.
static void lf_rows(const float* obs, int64_t lo, int64_t hi, int32_t obs_dim, double steer_gain, double throttle,
                    double bbox_half, double* out) {
    const double half = throttle * 0.5;
    for (int64_t r = lo; r < hi; ++r) {
        if (r + DG_LF_PREFETCH < hi) __builtin_prefetch(obs + (r + DG_LF_PREFETCH) * obs_dim + 2);
        const float* g = obs + r * obs_dim + 2;
        const double sn = double(g[0]), cs = double(g[1]), dist = double(g[2]) * bbox_half;
        double steer = steer_gain * sn;
        steer = steer < -1.0 ? -1.0 : steer;      // np.maximum(x, -1): NaN and -0.0 pass through
        steer = steer > 1.0 ? 1.0 : steer;        // np.minimum(x, 1)
        if (cs < 0.0) steer = sn >= 0.0 ? 1.0 : -1.0;
        out[3 * r] = dist > 5.0 ? throttle : half;
        out[3 * r + 1] = steer;
        out[3 * r + 2] = 0.0;
    }
}

static inline void cpu_relax() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
}

// Helper threads for the host LaneFollower: a batch's rows are cache misses on a
// slab the device just wrote, so one core is bound by its outstanding misses;
// kLfWorkers threads take equal row ranges beside the caller.  They spin ~1 ms
// after a batch (a loop calls the policy every few hundred us), then sleep.
struct LfPool {
    static constexpr int kLfWorkers = 3;
    std::atomic<unsigned> gen{0};
    std::atomic<int> done{0};
    std::mutex mu;
    std::condition_variable cv;
    const float* obs = nullptr;
    int64_t rows = 0;
    int32_t obs_dim = 0;
    double gain = 0, thr = 0, bh = 0;
    double* out = nullptr;

    void work(int id) {
        unsigned seen = 0;
        for (;;) {
            const auto t0 = std::chrono::steady_clock::now();
            unsigned g;
            while ((g = gen.load(std::memory_order_acquire)) == seen) {
                if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(1)) {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return gen.load(std::memory_order_acquire) != seen; });
                } else {
                    cpu_relax();
                }
            }
            seen = g;
            const int parts = kLfWorkers + 1;
            lf_rows(obs, rows * (id + 1) / parts, rows * (id + 2) / parts, obs_dim, gain, thr, bh, out);
            done.fetch_add(1, std::memory_order_acq_rel);
        }
    }
};

int dg_lane_follower_rows(const float* obs, int64_t rows, int32_t obs_dim, double steer_gain, double throttle,
                          double bbox_half, double* out) {
    if (!obs || !out || rows < 0 || obs_dim < 5) return fail(DG_EINVAL, "dg_lane_follower_rows: bad argument");
    static std::mutex call_mu;
    static LfPool* pool = nullptr;
    static pid_t pool_pid = 0;
    std::unique_lock<std::mutex> lk(call_mu, std::try_to_lock);
    if (rows < 2048 || !lk.owns_lock()) {            // small batches / a concurrent caller: this thread only
        lf_rows(obs, 0, rows, obs_dim, steer_gain, throttle, bbox_half, out);
        return DG_OK;
    }
    if (!pool || pool_pid != getpid()) {             // (a forked child has no helper threads: a new pool)
        pool = new LfPool;
        pool_pid = getpid();
        for (int i = 0; i < LfPool::kLfWorkers; ++i) std::thread(&LfPool::work, pool, i).detach();
    }
    pool->obs = obs;
    pool->rows = rows;
    pool->obs_dim = obs_dim;
    pool->gain = steer_gain;
    pool->thr = throttle;
    pool->bh = bbox_half;
    pool->out = out;
    pool->done.store(0, std::memory_order_relaxed);
    {
        std::lock_guard<std::mutex> g(pool->mu);
        pool->gen.fetch_add(1, std::memory_order_acq_rel);
    }
    pool->cv.notify_all();
    lf_rows(obs, 0, rows / (LfPool::kLfWorkers + 1), obs_dim, steer_gain, throttle, bbox_half, out);
    while (pool->done.load(std::memory_order_acquire) < LfPool::kLfWorkers) cpu_relax();
    return DG_OK;
}

int dg_launch_count(dg_engine* eng) { return eng ? eng->launches : 0; }

#ifdef DG_TICK_TIMERS
int dg_debug_tick_clocks(long long* host_out, int n_blocks, int reset) {
    const int n = n_blocks < 65536 ? n_blocks : 65536;
    cudaError_t e;
    if (reset) {
        static long long zeros[65536 * 48 / 64];
        e = cudaSuccess;
        for (int i = 0; i < 64 && e == cudaSuccess; ++i)
            e = cudaMemcpyToSymbol(g_tick_acc, zeros, sizeof(zeros), sizeof(zeros) * i);
    } else {
        e = cudaMemcpyFromSymbol(host_out, g_tick_acc, sizeof(long long) * 48 * n);
    }
    return e == cudaSuccess ? DG_OK : cuda_fail(e, "dg_debug_tick_clocks");
}
#endif

#ifdef DG_PHASE_TIMERS
int dg_debug_phase_clocks(long long* host_out, int n_blocks) {
    const int n = n_blocks < 65536 ? n_blocks : 65536;
    const cudaError_t e = cudaMemcpyFromSymbol(host_out, g_phase_clock, sizeof(long long) * 40 * n);
    return e == cudaSuccess ? DG_OK : cuda_fail(e, "dg_debug_phase_clocks");
}
#endif

int dg_tune(dg_engine* eng, int32_t mode, int32_t warps_per_world, int32_t ctas_per_sm) {
    if (!eng) return fail(DG_EINVAL, "dg_tune: null engine");
    if (mode == 1) {
        if (!eng->base.scratch) return fail(DG_EINVAL, "dg_tune: split mode needs the scratch buffer");
        const int apc = warps_per_world;
        if (apc != 2 && apc != 4 && apc != 8) return fail(DG_EINVAL, "dg_tune: split mode takes 2, 4 or 8 agents per CTA");
        const int blocks = ctas_per_sm > 0 ? ctas_per_sm : (apc == 2 ? 8 : apc == 4 ? 4 : 2);
        if (!has_split_variant(32 * apc, blocks)) return fail(DG_EINVAL, "dg_tune: no split kernel variant for this shape");
        eng->mode = 1;
        eng->warps_per_world = apc;
        eng->min_blocks = blocks;
        return DG_OK;
    }
    if (mode != 0 && mode != 2)
        return fail(DG_EINVAL, "dg_tune: mode must be 0 (fused), 1 (split) or 2 (fused, physics warp)");
    if (warps_per_world < 1 || warps_per_world > kMaxAgents)
        return fail(DG_EINVAL, "dg_tune: warps_per_world must lie in [1, 16]");
    const int nw = warps_per_world < eng->base.d.M ? warps_per_world : eng->base.d.M;
    const bool spec = mode == 2;
    if (spec && nw > 7) return fail(DG_EINVAL, "dg_tune: mode 2 takes at most 7 scan warps");
    const int threads = variant_threads(nw, spec);
    int blocks = ctas_per_sm > 0 ? ctas_per_sm : (threads == 512 ? 1 : threads >= 256 ? 2 : 4);
    if (!has_variant(threads, blocks, spec, eng->base.d.geometry_global != 0))
        return fail(DG_EINVAL, "dg_tune: no kernel variant for this shape");
    eng->warps_per_world = nw;
    eng->min_blocks = blocks;
    eng->mode = mode;
    return DG_OK;
}

size_t dg_scratch_bytes(int32_t W, int32_t M) { return split_scratch_bytes(W, M); }

int32_t dg_index_stride(dg_engine* eng) { return eng ? eng->base.index_stride : 0; }

}  // extern "C"
