/*
 * drivegrid_b200 -- C ABI of the B200 (sm_100a) batched vehicle step.
 *
 * The reference (/root/reference/pkg) is a Python package with no native
 * layer; the entry points below are what its engine/binding surface binds to
 * when the step runs on the GPU.  Each function names the reference interface
 * it replaces.  Plain C types only: no torch, no C++ in the signatures.
 *
 * Memory model: every device buffer in DgEngineDesc / DgStepIO is allocated by
 * the caller (the Python host uses torch tensors) and BORROWED by the engine
 * for its lifetime.  The library allocates nothing on the device.  All calls
 * are asynchronous on the given stream unless stated otherwise; calls on one
 * engine must be serialised by the caller (the reference is single-writer,
 * SPEC.md:377-379).
 *
 * Layouts (W worlds, M agents per world, row-major, C order):
 *   state      f64 [12][W][M]   field order of STATE_FIELDS (vehicle.py:124-142),
 *                               global coordinates exactly as the reference
 *   obs        f32 [W][M][D]    D = ego_dim + 5*k_road + 7*k_vehicles
 *   actions    f32|f64 [W][M][3]
 *   events     u8  [W][M][4]    goal, collision, crash, lane_forbidden (one-hot)
 *   terms      f64 [7][W][M]    progress, lane, offroad, idle, ttc_vehicle, ttc_edge, total
 */
#ifndef DRIVEGRID_B200_H
#define DRIVEGRID_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_ABI_VERSION 13
#define DG_NUM_STATE 12
#define DG_NUM_TERMS 7
#define DG_NO_ERROR 0x7fffffff

/* status codes (Python maps them to the reference's exception types) */
enum {
    DG_OK = 0,
    DG_EINVAL = 1,       /* bad argument / shape  -> ValueError                */
    DG_ENONFINITE = 2,   /* non-finite action      -> ValueError("non-finite action for world w agent m") */
    DG_ECUDA = 3,        /* CUDA runtime failure   -> RuntimeError             */
    DG_ENOSUPPORT = 4    /* configuration outside the kernel's limits          */
};

/* Integer dimensions and switches (engine.py:41-67, observation.py:18-35). */
typedef struct DgDims {
    int32_t W, M;
    int32_t obs_dim, ego_dim, k_road, k_vehicles, include_weather;
    int32_t dynamic;          /* 1 = 120 Hz single-track, 0 = 30 Hz bicycle */
    int32_t decimation;
    int32_t episode_len;
    int32_t invincible;
    int32_t collision_warmup;
    int32_t num_scenes;
    int32_t max_scene_bytes;  /* largest per-scene geometry blob, bytes      */
    int32_t max_segments;     /* largest P over scenes                       */
    int32_t geometry_global;  /* 0: scene blobs are per scene, in scene-local
                                 coordinates (the fused kernel stages its world's
                                 blob in shared memory by TMA and adds the grid
                                 offset); 1: blobs are per world, already moved
                                 by the offset, read in place from global memory
                                 by the fused kernel's global-geometry variants
                                 (modes 0 and 2, multi-tick) or the split
                                 kernels (mode 1: ticks = 1, written to ring
                                 slot ring_start) -- scenes too large for the
                                 227 KB of shared memory                       */
} DgDims;

/* Float64 scalars, precomputed on the host with the reference's expression
 * order (vehicle.py:237-336, observation.py, rewards.py:37-63). */
typedef struct DgConsts {
    double physics_dt, control_dt;
    double kp_steer, kd_steer, theta_max, tau_steer_max, steer_inertia, steer_limit;
    double a_f, b_r, tau_drive_max, tau_brake_front, tau_brake_rear, wheel_radius;
    double cornering_stiffness, f_z, chassis_mass, lambda_lat, lambda_yaw, yaw_inertia;
    double i_axle, wheelbase;
    double bic_a_max, bic_b_max, bic_c_roll, bic_steer_max;
    double road_radius, road_radius_sq, bbox_half, speed_norm, type_norm, ttc_max;
    double goal_radius, goal_weight, collision_weight, crash_weight, crash_drift_limit;
    double lane_forbidden_weight, progress_weight, progress_clamp, lane_weight, lane_sigma;
    double lane_heading_weight, lane_heading_base, offroad_weight, offroad_lat_limit;
    double offroad_dist_limit, idle_weight, idle_speed, ttc_vehicle_alpha, ttc_vehicle_pmax;
    double ttc_edge_alpha, ttc_edge_pmax, ttc_floor, edge_range, crash_speed_limit, offstage_x;
} DgConsts;

/* Engine description (replaces drivegrid.engine.Engine.__init__ tables,
 * engine.py:151-230).  Scene geometry is de-duplicated: worlds that share a
 * scene share one blob.  Per-scene blob, 16-byte aligned sections, local
 * coordinates:  f64x2 mid[P]; f64x2 dir[P]; f64 half_len[P]; f64 half_wid[P];
 * f32 type_feat[P] = float32(type / type_norm); lane subset f64x4
 * {mid, dir}[KL], f64 half_len[KL]; edge subset f64x2 mid[KE], i32 index[KE];
 * then the 64-byte spatial-index header of paper_2605_08528_b200/spatial.py;
 * that prefix is what the kernel copies to shared memory.  The index's
 * candidate lists follow in global memory.
 * scene_meta[s] = {byte_offset, smem_bytes, P, KL, KE, aux_offset, aux_bytes, 0}
 * (int64, byte offsets from scene_blob). */
typedef struct DgEngineDesc {
    DgDims dims;
    DgConsts k;
    const uint8_t* scene_blob;
    const int64_t* scene_meta;
    const int32_t* scene_of_world;  /* [W]        */
    const double* grid_offset;      /* [W][2]     */
    const double* mu_eff;           /* [W]        */
    const double* weather;          /* [W][4]     */
    const uint8_t* valid;           /* [W][M]     */
    const double* length;           /* [W][M]     */
    const double* width;            /* [W][M]     */
    const double* r_hull;           /* [W][M]     */
    const double* d_hull;           /* [W][M]     */
    double* state;                  /* [12][W][M] */
    uint8_t* alive;                 /* [W][M]     */
    int8_t* reason;                 /* [W][M]     */
    uint8_t* event_seen;            /* [W][M] bit k = EVENT_TYPES[k] latched */
    int32_t* spawn_step;            /* [W][M]     */
    int32_t* step_count;            /* [W]        */
    double* start_xy;               /* [W][M][2]  */
    double* goal_xy;                /* [W][M][2]  */
    double* start_yaw;              /* [W][M]     */
    int32_t* error_word;            /* [1] DG_NO_ERROR or first bad flat action index */
    uint8_t* scratch;               /* dg_scratch_bytes(W, M) bytes, or NULL (fused mode only) */
} DgEngineDesc;

/* Outputs of one control tick (StepOutput, engine.py:70-76, 397-406).
 * Optional pointers may be NULL. */
typedef struct DgStepIO {
    const void* actions;        /* [W][M][3]                                  */
    int32_t actions_f64;        /* 0: float32 actions, 1: float64             */
    int32_t autoreset;          /* 1: teleport_reset(dones) fused after the tail */
    float* obs;                 /* [W][M][D]   required                       */
    double* rewards;            /* [W][M]      required                       */
    uint8_t* dones;             /* [W][M]      required                       */
    uint8_t* events;            /* [W][M][4]   required                       */
    int8_t* reason_out;         /* [W][M]      info["reason"]                 */
    uint8_t* alive_out;         /* [W][M]      info["alive"] (before autoreset) */
    uint8_t* alive_pre_out;     /* [W][M]      info["alive_pre"]              */
    double* ttc_min_out;        /* [W][M]      info["ttc_min"]                */
    double* terms_out;          /* [7][W][M]   info["reward_terms"]           */
    double* snapshot_out;       /* [12][W][M]  info["state"] (pre-park)       */
    double* next_actions;       /* [W][M][3]   fused LaneFollower on this tick's
                                   observation (policies.py:21-43), or NULL  */
    double policy_gain, policy_throttle;
    uint32_t* event_counts;     /* [W][5]      += per-world counts of this tick's goal,
                                   collision, crash, lane_forbidden events and of
                                   alive agents (CASPS numerator), or NULL     */
    int32_t ticks;              /* control ticks in this launch (0/1: one step).  A
                                   T-tick launch equals T dg_step calls: tick t reads
                                   actions + t*W*M*3 -- or, when next_actions is set,
                                   the fused LaneFollower's actions of tick t-1 for
                                   t >= 1 (env.py:48-65 driven by policies.py:21-43) --
                                   and writes every per-tick output above at slot
                                   (ring_start + t) % ring_slots (obs + slot*W*M*D,
                                   rewards + slot*W*M, events + slot*W*M*4, ...).
                                   A rejected tick stops its world after the
                                   previous tick; error_word gets the flat index
                                   t*W*M*3 + w*M*3 + j.  Fused mode only.       */
    int32_t ring_slots;         /* 0: ticks                                    */
    int32_t ring_start;
    int32_t obs_resident;       /* 1: the obs slots are this engine's: beyond the
                                   prefix lengths prefix_out records for a slot
                                   (from the slot's previous use; zero after the
                                   caller zeroed the slot and its prefix entries)
                                   every float of a row is zero, so the kernel
                                   clears only the span between a row's old and
                                   new prefix instead of the whole block.
                                   Needs prefix_out with one entry set per obs
                                   slot; a recorded length past the block (e.g.
                                   0x7fff after the caller wrote the slot) clears
                                   the whole block.  Results do not depend on it.
                                   0: every block is cleared in full.  Fused
                                   modes; mode 1 ignores it.                   */
    double* drac_max;           /* [W][M]      episode safety metric, accumulated:
                                   drac_max = max(drac_max, pairwise DRAC of this
                                   tick's post-physics state over the agents alive
                                   before it) -- episode_metrics' per-agent max
                                   (metrics.py:33-62, 101-108), or NULL        */
    uint8_t* metric_seen;       /* [W][M]      |= bit 0 goal event, bit 1 collision
                                   event of this tick (metrics.py:100-101), or NULL */
    int32_t* index_out;         /* [W][M][dg_index_stride()] per tick slot, or NULL:
                                   the integer decisions behind the float outputs,
                                   for exact comparison with the reference --
                                   [0] nearest-lane index into the world's lane
                                       subset (rewards.py:94 argmin; -1: no lane or
                                       agent not alive before the tick),
                                   [1] road candidates kept n_r (observation.py:94-99),
                                   [2] valid neighbours n_v (observation.py:242-249),
                                   [3 .. 3+take_veh)  neighbour agent index by rank
                                       (stable argsort, observation.py:246), first n_v,
                                   [3+take_veh ..)    road slot -> segment index
                                       (stable argsort of ~cand), first n_r;
                                   entries past n_v / n_r are left untouched    */
    int16_t* prefix_out;        /* [W][M][2] per tick slot, or NULL: the length in
                                   floats of the part of each agent's road block
                                   (5 n_r) and vehicle block (7 n_v) that can be
                                   non-zero -- the rest of the row is zero
                                   (dg_to_host moves only these prefixes)      */
    uint64_t* phase_cycles;     /* [5] or NULL: device cycles spent per phase of
                                   the reference's phase_seconds (engine.py:33,
                                   342-395) -- action, physics, observation,
                                   reward_termination, reset -- summed over the
                                   warps that run them (lane 0 of each warp times
                                   its own segments), added to the 5 counters.
                                   Phases run concurrently on different warps,
                                   so they measure where the device work goes,
                                   not a wall-clock split.  Fused modes only.  */
} DgStepIO;

typedef struct dg_engine dg_engine;

/* Engine lifetime (Engine.__init__ / garbage collection). */
int dg_create(const DgEngineDesc* desc, dg_engine** out);
int dg_destroy(dg_engine* eng);

/* One 30 Hz control tick for every world: Engine.step (engine.py:334-406),
 * EnvHandle.step (env.py:48-65).  Worlds whose actions contain a non-finite
 * value are not stepped; their first bad flat index is min-reduced into
 * error_word (engine.py:286-295 raises before mutating; the host obtains
 * that exact behaviour with dg_check_actions + dg_read_error first). */
int dg_step(dg_engine* eng, const DgStepIO* io, void* stream);

/* Observation of the current state without stepping: Engine.observe
 * (engine.py:297-330); optional fused LaneFollower actions as in DgStepIO. */
int dg_observe(dg_engine* eng, float* obs, double* ttc_min_out, double* next_actions, double policy_gain,
               double policy_throttle, void* stream);

/* Masked teleport reset: Engine.teleport_reset (engine.py:599-619).
 * mask [W][M] u8 (NULL = every valid slot); optional new starts/goals
 * [W][M][2] and headings [W][M] (device, global coordinates). */
int dg_reset(dg_engine* eng, const uint8_t* mask, const double* new_starts,
             const double* new_goals, const double* new_headings, void* stream);

/* Copy of the 12-field state [12][W][M] f64 out of / into the engine
 * (Engine.state / set_state; the teacher-forced parity harness).  `dst` /
 * `src` may be host (pinned or pageable) or device memory; asynchronous on
 * stream for device and pinned memory. */
int dg_get_state(dg_engine* eng, double* dst, void* stream);
int dg_set_state(dg_engine* eng, const double* src, void* stream);

/* step_count assignment (EnvHandle.reset sets it to 0, env.py:42). */
int dg_set_step_count(dg_engine* eng, int32_t value, void* stream);

/* Finiteness scan of an action batch into error_word (engine.py:291-294). */
int dg_check_actions(dg_engine* eng, const void* actions, int32_t actions_f64, void* stream);

/* Synchronising read of error_word; resets it.  *flat_index = -1 if clean. */
int dg_read_error(dg_engine* eng, int32_t* flat_index, void* stream);

/* Device LaneFollower (policies.py:21-43): obs [W][M][D] -> float64 actions
 * [W][M][3], the same values the host numpy policy produces. */
int dg_lane_follower(dg_engine* eng, const float* obs, double* actions, double steer_gain,
                     double throttle, void* stream);

/* Pairwise DRAC of logged states (metrics.py:33-62 pairwise_drac, applied per
 * record by episode_metrics, metrics.py:86-125), no engine needed.
 * x, y, yaw, v_x, v_y, alive: [steps][W][M]; v_x/v_y are the body-frame
 * velocity of STATE_FIELDS (rotated by yaw as metrics.py:104-107 does) or,
 * with world_velocity != 0, pairwise_drac's vel_world argument as is;
 * r_hull, d_hull: [W][M].  out [W][M] = max over the steps of each record's
 * per-agent max DRAC, also max'ed with the incoming out when accumulate != 0.
 * M <= 16.  Device pointers; asynchronous on stream. */
int dg_pairwise_drac(const double* x, const double* y, const double* yaw, const double* v_x,
                     const double* v_y, const uint8_t* alive, const double* r_hull,
                     const double* d_hull, int32_t steps, int32_t W, int32_t M, double* out,
                     int32_t accumulate, int32_t world_velocity, void* stream);

/* Batched system-identification rollouts (sysid.py:201-228 rollout_channels,
 * evaluated for every candidate x maneuver of a CEM generation at once):
 * consts [B] DgConsts (device, one per candidate parameter vector, built like
 * dg_create's), mu [B][3] effective friction per surface (dry, wet, gravel),
 * tick_start [n_maneuvers + 1] offsets into actions [ticks][3] (decoded
 * throttle / steer / brake per 30 Hz tick) and surface [ticks] (0..2);
 * out + out_offset[m] receives maneuver m's channels [7][2 * ticks_m][B]
 * (x, y, yaw, speed, yaw_rate, wheel_speed, steer_angle at 60 Hz). */
int dg_sysid_rollout(const void* consts, const double* mu, const int32_t* tick_start, const double* actions,
                     const uint8_t* surface, const int64_t* out_offset, int32_t B, int32_t n_maneuvers,
                     double* out, void* stream);

/* Host delivery of one step's outputs (the numpy path of Engine.step /
 * observe, engine.py:297-335, env.py:48-65).  dg_host_alloc returns zeroed,
 * mapped, portable pinned host memory (cudaHostAlloc); dg_host_free releases it.
 * dg_to_host writes the engine's device observation `obs` [W][M][D] into
 * such a slab `host_obs` (same layout) so that the slab equals it bit for
 * bit, moving only the non-zero prefix of every row's road and vehicle blocks
 * over PCIe -- the lengths come from `prefix` (the step's DgStepIO.prefix_out)
 * or, when it is NULL, from a scan for the last non-zero float (bitwise);
 * `prev_len` (device int32 [W*M][2], zero for a fresh slab) holds
 * the prefix lengths the slab currently carries and is updated.  Then
 * `aux_bytes` of the packed per-tick outputs `aux` (device) are copied to
 * `host_aux` (pinned).  `bytes` (device u64, optional) accumulates the
 * observation bytes written to the host.  Async on `stream`; the slab is valid
 * after the stream synchronises. */
int dg_host_alloc(size_t bytes, void** host_ptr);
int dg_host_free(void* host_ptr);
int dg_to_host(dg_engine* eng, const float* obs, const int16_t* prefix, float* host_obs, int32_t* prev_len,
               const void* aux, void* host_aux, size_t aux_bytes, unsigned long long* bytes, void* stream);

/* The numpy step path in one host call (replaces the four calls of
 * Engine._step_host: the host finiteness check engine.py:291-294, the action
 * H2D copy, dg_step, dg_to_host; engine.py:334-406 behind env.py:48-65).
 * host_actions: the caller's float64 [W][M][3] (any host memory); checked for
 * finiteness while copied into pinned_actions (pinned, same size) -- a
 * non-finite value returns DG_ENONFINITE with *bad_index = its flat index,
 * before anything is queued or mutated; else *bad_index = -1.  Then, on
 * `stream`: pinned_actions -> io->actions (device, io->actions_f64 = 1), the
 * step of `io`, and -- when host_obs is non-NULL -- dg_to_host(io->obs,
 * io->prefix_out, host_obs, prev_len, aux, host_aux, aux_bytes, bytes). */
int dg_step_host(dg_engine* eng, const DgStepIO* io, const double* host_actions, double* pinned_actions,
                 float* host_obs, int32_t* prev_len, const void* aux, void* host_aux, size_t aux_bytes,
                 unsigned long long* bytes, int64_t* bad_index, void* stream);

/* Host LaneFollower (policies.py:21-43) over float32 observation rows
 * obs [rows][obs_dim] (host memory) -> out [rows][3] float64 (throttle, steer,
 * brake): bit-identical to the numpy policy (NaN and -0.0 included).  Host
 * code, no device work. */
int dg_lane_follower_rows(const float* obs, int64_t rows, int32_t obs_dim, double steer_gain, double throttle,
                          double bbox_half, double* out);

/* Kernel launches issued by the last dg_step/dg_observe/dg_reset call. */
int dg_launch_count(dg_engine* eng);

/* Launch shape -- a performance knob only, results do not depend on it.
 *   mode 0 (fused): one CTA per world, warps_per_world warps (1..16; agents
 *                   strided over the warps)
 *   mode 1 (split): a physics kernel (one warp per world) chained by
 *                   programmatic dependent launch to a per-agent kernel with
 *                   warps_per_world (2, 4 or 8) agents per CTA; needs scratch
 *   mode 2 (fused, physics warp): mode 0 with warps_per_world (<= 8) scan
 *                   warps plus one warp that runs tick t + 1's physics while
 *                   the others build tick t's observation (multi-tick launches)
 * ctas_per_sm selects the register budget of the kernel variant (0 = default). */
int dg_tune(dg_engine* eng, int32_t mode, int32_t warps_per_world, int32_t ctas_per_sm);

/* Device scratch the split mode needs (per-agent records between its kernels). */
size_t dg_scratch_bytes(int32_t W, int32_t M);

/* int32 entries per agent of DgStepIO.index_out: 3 + min(k_vehicles, M) +
 * min(k_road, max_segments). */
int32_t dg_index_stride(dg_engine* eng);

/* ------------------------------------------------------------------------
 * Policy MLP (BASELINE configs[4]: the rollout's batched policy forward,
 * fused into the env loop on the device).  The reference has no policy code;
 * the network is the paper's App. E: per-net ego
 * 11->64->64, road 5->96->96 and vehicle 7->96->96 encoders with masked
 * max-pool over the observation's valid slots, trunk 256->128->64 (ELU),
 * actor head 64->3 (mean), critic head 64->1; actor and critic do not share
 * weights.  Runs on tcgen05 tensor cores (bf16 operands, fp32 accumulate).
 *
 * Weights: one blob per net (net 0 = actor, 1 = critic), net n at
 * weights + n * net_stride; off[] = byte offsets of the sections below inside
 * a net's blob (16-byte aligned).  W_* sections are bf16 tiles [out][in] in
 * the canonical K-major UMMA layout (8x8 core matrices, element (r, k) at
 * ((r/8)*(K/8) + k/8)*128 + (r%8)*16 + (k%8)*2, K = in padded to 16 for the
 * first layers); B_* and W_HEAD / B_HEAD are float32 (W_HEAD [out][64]). */
enum {
    DG_POL_W_EGO1 = 0, DG_POL_W_EGO2, DG_POL_W_T1, DG_POL_W_T2,
    DG_POL_W_ROAD1, DG_POL_W_ROAD2, DG_POL_W_VEH1, DG_POL_W_VEH2,
    DG_POL_B_EGO1, DG_POL_B_EGO2, DG_POL_B_ROAD1, DG_POL_B_ROAD2, DG_POL_B_VEH1, DG_POL_B_VEH2,
    DG_POL_B_T1, DG_POL_B_T2, DG_POL_W_HEAD, DG_POL_B_HEAD,
    DG_POL_LOG_STD,             /* actor only: float32 [4] (3 used), the state-independent log sigma */
    DG_POL_NUM_SECTIONS
};

typedef struct DgPolicyDesc {
    int32_t n_agents;           /* rows of obs (W * M)                              */
    int32_t obs_dim, ego_dim, k_road, k_vehicles;
    int32_t critic;             /* 1: also run net 1 (value head)                   */
    const float* obs;           /* [n_agents][obs_dim] float32, device              */
    const uint8_t* weights;     /* net blobs, device                                */
    int64_t net_stride;
    int64_t off[DG_POL_NUM_SECTIONS];
    uint16_t* emb;              /* scratch: dg_policy_scratch_bytes(n_agents, nets)  */
    float* mean;                /* [n_agents][3] actor mean, or NULL                */
    double* actions;            /* [n_agents][3] the same mean as float64 env actions
                                   (the next tick's input), or NULL                */
    float* value;               /* [n_agents] critic value, or NULL                 */
    int32_t sample;             /* 0: actions = the actor mean; 1: PPO sampling,
                                   actions = mean + exp(log_std) * eps with eps ~ N(0, 1)
                                   from Philox4x32-10 (key = seed, counter = {agent
                                   index, counter}) and Box-Muller in float64        */
    int32_t first_net;          /* 0: nets 0 (actor) [and 1 with critic]; 1: the critic alone --
                                   a trainer can run the value head on a side stream */
    uint64_t seed;
    uint64_t counter;           /* e.g. the rollout tick: a fresh draw per tick      */
    float* log_prob;            /* [n_agents] log pi(actions | obs) (diagonal Gaussian), or NULL */
    float* actions_f32;         /* [n_agents][3] the written actions as float32 (the
                                   rollout's action record), or NULL                */
    const int16_t* prefix;      /* [n_agents][2] the step's DgStepIO.prefix_out for these
                                   rows (5 n_r, 7 n_v: the valid road / vehicle slots of
                                   each observation row), or NULL: the encoder finds the
                                   counts by scanning the rows                        */
    int32_t* work_counter;      /* [2] zero-initialised int32 (device), or NULL: the
                                   encoder's work queue -- persistent CTAs take (net,
                                   agent group, modality) items by one atomic each;
                                   entry first_net is used and reset to 0 by the
                                   forward's second kernel, so one buffer serves every
                                   forward on a stream (an actor-only and a
                                   critic-only forward may run concurrently).  NULL:
                                   one CTA per (agent group, net)                   */
} DgPolicyDesc;

/* One forward of the policy over every agent's observation row: 2 kernel
 * launches (encoders, trunk + heads), asynchronous on stream. */
int dg_policy_forward(const DgPolicyDesc* desc, void* stream);
size_t dg_policy_scratch_bytes(int32_t n_agents, int32_t nets);

/* Generalised advantage estimation over a rollout of T transitions for N
 * agents (the PPO batch of BASELINE configs[4]): with
 * done_t = the transition ended the episode,
 *   delta_t = r_t + gamma * V_{t+1} * (1 - done_t) - V_t
 *   A_t     = delta_t + gamma * lambda * (1 - done_t) * A_{t+1}
 * rewards [T][N] f64, dones [T][N] u8, values [T+1][N] f32 (row T = bootstrap);
 * advantages, returns (= A + V) [T][N] f32.  Float64 accumulation. */
int dg_gae(const double* rewards, const uint8_t* dones, const float* values, int32_t T, int64_t N,
           double gamma, double lambda, float* advantages, float* returns, void* stream);
const char* dg_policy_last_error(void);

/* ------------------------------------------------------------------------
 * On-device world construction.  Replaces the reference's
 * O(W) Python init: build_world_batch (world.py:82-194 -- segmentize,
 * scene_segments, grid_offsets, assign_scenes, the padded (W, P_max)
 * arrays), the Engine spawn table (engine.py:192-227 with filter_agents,
 * scenario.py:169-192), Engine._compact_subset (engine.py:234-253) and
 * eval.random_goals (resample_goal / polyline_arc_point,
 * config.py:222-278).  The host keeps scene intake (JSON, recentre, z-flatten,
 * degeneracy verdicts, config.py:162-189), the Philox draws (the scene-order
 * permutation of assign_scenes, the goal distances) and weather / friction.
 * Every output is bit-identical to the reference. */

/* The prepared scene pool, flattened (device arrays). */
typedef struct DgScenePool {
    int32_t num_scenes, num_polylines, num_points, num_agents;
    const double* points;        /* [num_points][2] polyline vertices x, y (scene-local,
                                    recentred), polyline after polyline, scene after scene */
    const int32_t* poly_start;   /* [num_polylines + 1] first vertex of each polyline       */
    const int32_t* poly_type;    /* [num_polylines] type code                               */
    const int32_t* scene_poly;   /* [num_scenes + 1] first polyline of each scene           */
    const double* agents;        /* [num_agents][7] start x, start y, start heading, goal x,
                                    goal y, length, width -- file order within a scene      */
    const int32_t* scene_agent;  /* [num_scenes + 1] first agent record of each scene       */
} DgScenePool;

typedef struct DgSceneBuild {
    double gap;                  /* segment_gap (SEGMENT_GAP 3.0)                           */
    double bbox_half;            /* scene_factory.bbox_half                                 */
    double half_width;           /* SEGMENT_HALF_WIDTH (0.05)                               */
    double goal_radius;          /* filter_agents' start-goal threshold                     */
    int32_t cap;                 /* agents kept per scene (num_agents_per_env)              */
    int32_t pad_;
} DgSceneBuild;

/* Per-scene tables (device, caller-allocated).  Scene s owns the rows from
 * base(s) = poly_start[scene_poly[s]] - scene_poly[s] (its first candidate pair)
 * on: segments [base, base + seg_count[s]) in scene_segments order, lane / edge
 * index lists (scene-local segment indices, ascending) at lane_index + base /
 * edge_index + base.  Arrays marked [pairs] hold num_points - num_polylines rows. */
typedef struct DgSceneSegments {
    double* mid;                 /* [pairs][2] 0.5 * (a + b)                                */
    double* dir;                 /* [pairs][2] (b - a) / |b - a|                            */
    int32_t* type;               /* [pairs]                                                  */
    double* half_len;            /* [pairs] 0.5 * |b - a|                                   */
    double* half_wid;            /* [pairs] half_width                                      */
    int32_t* lane_index;         /* [pairs]                                                  */
    int32_t* edge_index;         /* [pairs]                                                  */
    double* arc;                 /* [num_points] cumulative arc length at each vertex of
                                    its polyline (np.cumsum order)                          */
    int32_t* seg_count;          /* [num_scenes]                                             */
    int32_t* lane_count;         /* [num_scenes]                                             */
    int32_t* edge_count;         /* [num_scenes]                                             */
    int32_t* lane_polys;         /* [num_scenes] lane polylines of the scene                */
    int32_t* kept_count;         /* [num_scenes] filter_agents(scene, cap) length           */
    int32_t* kept_agent;         /* [num_agents] scene s: kept_agent[scene_agent[s] + k] =
                                    pool index of its k-th kept agent                       */
} DgSceneSegments;

/* Scene tables for a pool: one CTA per scene (3 passes: ordered segment
 * compaction, arc tables, spawn filter).  Asynchronous on stream. */
int dg_build_scenes(const DgScenePool* pool, const DgSceneBuild* build, DgSceneSegments* out, void* stream);

/* World w of this build is world world_base + w of the batch (a rank's shard
 * builds only its own worlds): scene scene_order[(world_base + w) % num_scenes]
 * (assign_scenes: the Philox permutation for random_fill, the identity for
 * fixed), grid offset ((g % grid_cols) * pitch, (g / grid_cols) * pitch) with
 * g = world_base + w and grid_cols = ceil(sqrt(total worlds)). */
typedef struct DgWorldBuild {
    int32_t W, M, num_scenes, grid_cols;
    int64_t world_base;
    double pitch, offstage_x, wheelbase;
    const int32_t* scene_order;  /* [num_scenes]                                           */
    /* engine tables (required) */
    int32_t* assignment;         /* [W]                                                     */
    double* grid_offset;         /* [W][2]                                                  */
    uint8_t* valid;              /* [W][M]                                                  */
    uint8_t* alive;              /* [W][M] = valid, or NULL                                 */
    double* start_xy;            /* [W][M][2] global                                        */
    double* goal_xy;             /* [W][M][2] global                                        */
    double* start_yaw;           /* [W][M]                                                  */
    double* length;              /* [W][M] (4.0 in empty slots)                             */
    double* width;               /* [W][M] (2.0 in empty slots)                             */
    double* r_hull;              /* [W][M] circle_layout (observation.py:44-48)             */
    double* d_hull;              /* [W][M]                                                  */
    double* state;               /* [12][W][M] initial state (parked empty slots)           */
    /* eval.random_goals: goal_min == goal_max walks exactly goal_min; else
       goal_draws [draws] holds rng.uniform(goal_min, goal_max) of Philox stream
       (seed, 4), one per valid agent of a scene with lanes, in (world, agent)
       order over the whole batch (world 0 first, also for a shard) */
    int32_t random_goals, pad_;
    double goal_min, goal_max;
    const double* goal_draws;
    /* padded WorldBatch (p_max > 0; world.py:148-194) [W][p_max](..) */
    int32_t p_max, k_lane, k_edge, pad2_;
    double* wb_mid;              /* [W][p_max][2] scene-local                               */
    double* wb_dir;
    int32_t* wb_type;
    double* wb_half_len;
    double* wb_half_wid;
    uint8_t* wb_mask;
    /* _compact_subset (k_lane / k_edge > 0): [W][K](..), midpoints global */
    double* lane_mid;
    double* lane_dir;
    double* lane_half_len;
    double* lane_half_wid;
    uint8_t* lane_mask;
    double* edge_mid;
    double* edge_dir;
    double* edge_half_len;
    double* edge_half_wid;
    uint8_t* edge_mask;
} DgWorldBuild;

/* Per-world tables of a batch from dg_build_scenes' output: one thread per
 * (world, agent) slot (spawn table + initial state, then the goal walk) and
 * per (world, segment) / (world, k) for the optional padded and subset
 * arrays.  Asynchronous on stream. */
int dg_build_worlds(const DgScenePool* pool, const DgSceneSegments* scenes, const DgWorldBuild* build,
                    void* stream);

const char* dg_last_error(void);
int dg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DRIVEGRID_B200_H */
