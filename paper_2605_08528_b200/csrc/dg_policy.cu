// dg_policy.cu -- the batched actor-critic policy MLP of SceneFactory
// (arXiv 2605.08528, App. E) on tcgen05 tensor cores,
// reading the step kernel's observation rows in place (BASELINE configs[4]:
// the rollout's policy forward fused into the env loop, no host round trip).
//
// Network (per net; the actor and the critic have separate weights):
//   ego      11 -> 64 -> 64                  ELU, ELU
//   road      5 -> 96 -> 96  per point       ELU, ELU, masked max-pool over the K_r slots
//   vehicle   7 -> 96 -> 96  per neighbour   ELU, ELU, masked max-pool over the K_v slots
//   trunk   256 -> 128 -> 64                 ELU, ELU   (concat ego | road | vehicle)
//   head     64 -> 3 (actor mean) or 1 (critic value), linear
//
// Masked max-pool only ever sees valid slots: the observation's road and
// vehicle blocks are prefix-compacted (observation.py:98-124, 242-293), so a
// world's valid points are the first n of each agent.  Each agent's points are
// packed into 8-row segments (the last one padded with copies of the agent's
// first point, which cannot change a max), 16 segments per 128-row tcgen05
// tile; the per-segment max is an 8-lane shuffle reduction of the TMEM rows
// and agents combine their segments with ordered-integer atomicMax in shared
// memory.  max commutes with the monotone ELU(x + b), so the pool runs on the
// raw layer-2 accumulator and the bias + ELU is applied once per agent.  An
// agent with no valid slot gets a zero embedding.
//
// Kernels (two launches per forward; grid.y = net):
//   policy_encoder_kernel  64 agents per CTA: road and vehicle encoders,
//                          L1 (K padded to 16) and L2 (K = 96) as tcgen05 GEMMs
//                          with M = 128 point rows, TMEM accumulators
//   policy_trunk_kernel    128 agents per CTA: ego encoder, trunk, head
// Operands are bf16 in canonical K-major shared-memory tiles (dg_umma.cuh),
// accumulation fp32 in TMEM; biases, ELU, max and the head in fp32.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>

#include "dg_umma.cuh"
#include "drivegrid_b200.h"

namespace {

#ifndef DG_ENC_AGENTS
#define DG_ENC_AGENTS 32
#endif
#ifndef DG_L2_NOSEL
#define DG_L2_NOSEL 1
#endif
#ifndef DG_ENC_CTAS_PER_SM
#define DG_ENC_CTAS_PER_SM 3
#endif
constexpr int kEncAgents = DG_ENC_AGENTS;   // agents per encoder CTA (<= 32: one per lane in the scan)
constexpr int kTrunkAgents = 128;  // agents per trunk CTA (one TMEM lane each)
constexpr int kHid = 96;           // road / vehicle encoder width
constexpr int kEgo = 64;
constexpr int kT1 = 128, kT2 = 64;
constexpr int kEmb = 2 * kHid;     // pooled road | vehicle, bf16, per agent and net

__device__ __forceinline__ float elu(float x) { return x > 0.0f ? x : __expf(x) - 1.0f; }

constexpr float kLog2e = 1.4426950408889634f;
// log2(e) * ELU(y / log2(e)): the encoders' first layers carry a log2(e) factor
// in their weights and bias (policy.py, fold_first_layer), so the exponential is
// one ex2 and the scale folds into one FFMA; the next layer's weights carry ln 2.
__device__ __forceinline__ float elu_log2(float y) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(y));
    return y > 0.0f ? y : fmaf(e, kLog2e, -kLog2e);
}

#ifdef DG_EXP_ELU2
__device__ __forceinline__ uint32_t elu_log2_bf16x2(float lo, float hi) {
    const uint32_t y = umma::pack_bf16(lo, hi);
    uint32_t m, e, r, o;
    asm("min.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(y), "r"(0u));
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(e) : "r"(m));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(e), "r"(0x3FB93FB9u), "r"(0xBFB9BFB9u));
    asm("max.bf16x2 %0, %1, %2;" : "=r"(o) : "r"(y), "r"(r));
    return o;
}
#endif

// float <-> order-preserving unsigned (0 = "no value yet")
__device__ __forceinline__ uint32_t f2o(float x) {
    const uint32_t b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// 16 consecutive bf16 of row r, columns c..c+15, of a canonical tile with K columns
__device__ __forceinline__ void store_row16(uint8_t* tile, int r, int c, int K, const float* v) {
    uint4 lo, hi;
    lo.x = umma::pack_bf16(v[0], v[1]);   lo.y = umma::pack_bf16(v[2], v[3]);
    lo.z = umma::pack_bf16(v[4], v[5]);   lo.w = umma::pack_bf16(v[6], v[7]);
    hi.x = umma::pack_bf16(v[8], v[9]);   hi.y = umma::pack_bf16(v[10], v[11]);
    hi.z = umma::pack_bf16(v[12], v[13]); hi.w = umma::pack_bf16(v[14], v[15]);
    *reinterpret_cast<uint4*>(tile + umma::kmajor_offset(r, c, K)) = lo;
    *reinterpret_cast<uint4*>(tile + umma::kmajor_offset(r, c + 8, K)) = hi;
}

__device__ __forceinline__ const uint8_t* net_base(const DgPolicyDesc& p, int net) {
    return p.weights + int64_t(net) * p.net_stride;
}
__device__ __forceinline__ const float* fsec(const DgPolicyDesc& p, int net, int which) {
    return reinterpret_cast<const float*>(net_base(p, net) + p.off[which]);
}

// ------------------------------------------------------------------ encoder
// Shared memory (bytes): A0 128x16 bf16 | A1 128x96 bf16 | W1 96x16 | W2 96x96 |
// acc u32[32][97] | cnt[32] | segstart[36] | seg u16[32 * ceil(K/8)] | bars
constexpr int kEncThreads = 256;   // 8 warps: lane quarter = warp % 4, column half = warp / 4
constexpr int kAccStride = kHid + 1;
struct EncSmem {
    static constexpr int kA0 = 0;
    static constexpr int kA1 = kA0 + 128 * 16 * 2;
    static constexpr int kW1 = kA1 + 128 * kHid * 2;
    static constexpr int kW2 = kW1 + kHid * 16 * 2;
    static constexpr int kAcc = kW2 + kHid * kHid * 2;
    static constexpr int kCnt = kAcc + kEncAgents * kAccStride * 4;
    static constexpr int kSegStart = kCnt + kEncAgents * 4;
    static constexpr int kB2 = kSegStart + (kEncAgents + 4) * 4;
    static constexpr int kSeg = kB2 + kHid * 4;
};

__host__ __device__ __forceinline__ int enc_seg_cap(int k_slots) { return kEncAgents * ((k_slots + 7) / 8); }
__host__ __device__ __forceinline__ size_t enc_smem_bytes(int k_max) {
    return size_t(EncSmem::kSeg) + ((size_t(enc_seg_cap(k_max)) * 2 + 15) & ~size_t(15)) + 64;
}

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(umma::smem_u32(bar)), "r"(bytes) : "memory");
}
// TMA bulk copy global -> shared, completing on bar (after expect_tx of the total)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(umma::smem_u32(dst)), "l"(src), "r"(bytes), "r"(umma::smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kEncThreads, 3) policy_encoder_kernel(const DgPolicyDesc p) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ int s_item;
    uint8_t* A0 = sm + EncSmem::kA0;
    uint8_t* A1 = sm + EncSmem::kA1;
    uint8_t* W1 = sm + EncSmem::kW1;
    uint8_t* W2 = sm + EncSmem::kW2;
    uint32_t* acc = reinterpret_cast<uint32_t*>(sm + EncSmem::kAcc);
    int* cnt = reinterpret_cast<int*>(sm + EncSmem::kCnt);
    int* segstart = reinterpret_cast<int*>(sm + EncSmem::kSegStart);
    uint16_t* seg = reinterpret_cast<uint16_t*>(sm + EncSmem::kSeg);
    float* b2 = reinterpret_cast<float*>(sm + EncSmem::kB2);
    const int kmax = p.k_road > p.k_vehicles ? p.k_road : p.k_vehicles;
    uint8_t* tail = sm + EncSmem::kSeg + ((enc_seg_cap(kmax) * 2 + 15) & ~15);
    uint64_t* bar = reinterpret_cast<uint64_t*>(tail);          // [0] MMA, [1] weights
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tail + 16);

    if (warp == 0) umma::tmem_alloc(tmem_slot, 128);
    if (tid == 32) {
        umma::bar_init(bar, 1);
        umma::bar_init(bar + 1, 1);
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *tmem_slot;     // D1 and D2 share columns 0..95 (D1 is drained before MMA2)
    // epilogue mapping: TMEM lane quarter q (rows 32q..32q+31), column half hf (48 columns)
    const int q = warp & 3, hf = warp >> 2;
    const int r = 32 * q + lane;                       // this thread's tile row
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const int c0 = 48 * hf;
    uint32_t phase = 0;
    uint32_t wphase = 0;           // parity of the weights barrier (one TMA load per item)
    const int nets = p.first_net == 1 ? 1 : (p.critic ? 2 : 1);
    const int n_groups = (p.n_agents + kEncAgents - 1) / kEncAgents;
    const int n_items = 2 * nets * n_groups;
    int step = 0;

    // Work items (net, agent group, modality).  With the work queue (persistent
    // CTAs, about three per SM): the road items (twice the tiles) first, then the
    // vehicle items, handed out by one atomic per item -- no tail of idle SMs
    // behind the last wave.  Without: this CTA's group of its net, both modalities.
    for (;;) {
        int net, g, mod;
        if (p.work_counter) {
            if (tid == 0) s_item = atomicAdd(p.work_counter + p.first_net, 1);
            __syncthreads();
            const int item = s_item;
            if (item >= n_items) break;
            mod = item / (nets * n_groups);
            const int rem = item - mod * nets * n_groups;
            net = p.first_net + rem / n_groups;
            g = rem - (rem / n_groups) * n_groups;
        } else {
            if (step == 2) break;
            mod = step;
            net = blockIdx.y + p.first_net;
            g = blockIdx.x;
        }
        ++step;
        const int a0 = g * kEncAgents;
        const int na = min(kEncAgents, p.n_agents - a0);
        const uint8_t* wb = net_base(p, net);
        const int nf = mod == 0 ? 5 : 7;
        const int kslots = mod == 0 ? p.k_road : p.k_vehicles;
        const int fbase = mod == 0 ? p.ego_dim : p.ego_dim + 5 * p.k_road;
        const int w1 = mod == 0 ? DG_POL_W_ROAD1 : DG_POL_W_VEH1;
        const int w2 = mod == 0 ? DG_POL_W_ROAD2 : DG_POL_W_VEH2;
        const float* gb2 = fsec(p, net, mod == 0 ? DG_POL_B_ROAD2 : DG_POL_B_VEH2);

        // weights of this modality: TMA bulk copies (the previous modality's MMAs are done)
        if (tid == 0) {
            expect_tx(bar + 1, kHid * 16 * 2 + kHid * kHid * 2);
            bulk_g2s(W1, wb + p.off[w1], kHid * 16 * 2, bar + 1);
            bulk_g2s(W2, wb + p.off[w2], kHid * kHid * 2, bar + 1);
        }
        for (int i = tid; i < kEncAgents * kAccStride; i += kEncThreads) acc[i] = 0u;
        for (int i = tid; i < kHid; i += kEncThreads) b2[i] = __ldg(gb2 + i);

        // valid slot counts (the valid slots are a prefix): from the step's prefix
        // record when given, else warp w probes agents 4w..4w+3, 64 slots per round
        // (two per lane), all eight loads per lane in flight together
        if (p.prefix) {
            for (int a = tid; a < na; a += kEncThreads) {
                const int v = int(__ldg(p.prefix + 2 * int64_t(a0 + a) + mod)) / nf;
                cnt[a] = v < kslots ? v : kslots;
            }
        } else {
            int c4[4] = {0, 0, 0, 0};
            bool more[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) more[j] = 4 * warp + j < na;
            for (int s0 = 0; s0 < kslots; s0 += 64) {
                bool ok[4][2];
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int s = s0 + 32 * h + lane;
                        ok[j][h] = false;
                        if (more[j] && s < kslots) {
                            const float* f = p.obs + int64_t(a0 + 4 * warp + j) * p.obs_dim + fbase + s * nf;
                            ok[j][h] = mod == 0 ? (__ldg(f + 3) != 0.0f || __ldg(f + 4) != 0.0f)
                                                : (__ldg(f + 2) != 0.0f);
                        }
                    }
                bool any = false;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const unsigned b0 = __ballot_sync(0xffffffffu, ok[j][0]);
                    const unsigned b1 = __ballot_sync(0xffffffffu, ok[j][1]);
                    if (more[j]) {
                        c4[j] += __popc(b0) + (b0 == 0xffffffffu ? __popc(b1) : 0);
                        more[j] = b0 == 0xffffffffu && b1 == 0xffffffffu;
                    }
                    any |= more[j];
                }
                if (!any) break;
            }
            if (lane < 4 && 4 * warp + lane < na) cnt[4 * warp + lane] = c4[0] * (lane == 0) + c4[1] * (lane == 1) +
                                                                        c4[2] * (lane == 2) + c4[3] * (lane == 3);
        }
        __syncthreads();
        if (warp == 0) {
            // exclusive scan of the per-agent segment counts (one agent per lane)
            const int n0 = lane < na ? (cnt[lane] + 7) >> 3 : 0;
            int incl = n0;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane <= na) segstart[lane] = incl - n0;
            if (lane == 31 && na == kEncAgents) segstart[kEncAgents] = incl;
        }
        __syncthreads();
        const int S = segstart[na];
        for (int a = warp; a < na; a += kEncThreads / 32) {
            const int s0 = segstart[a], n = segstart[a + 1] - s0;
            for (int j = lane; j < n; j += 32) seg[s0 + j] = uint16_t((a << 8) | j);
        }
        __syncthreads();

        // features of row r for the tile starting at segment t0 (warps 0-3 build A0)
        auto fetch = [&](int t0, float* f) {
            const int s = t0 + (r >> 3);
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = 0.0f;
            if (hf == 0 && s < S) {
                const int e = seg[s];
                const int a = e >> 8;
                int slot = 8 * (e & 255) + (r & 7);
                if (slot >= cnt[a]) slot = 0;                   // duplicate of a valid point
                const float* src = p.obs + int64_t(a0 + a) * p.obs_dim + fbase + slot * nf;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (i < nf) f[i] = __ldg(src + i);
                    if (i == nf) f[i] = 1.0f;                   // bias column of W1
                }
            }
        };
        float fcur[8];
        fetch(0, fcur);
        for (int t0 = 0; t0 < S; t0 += 16) {
            const int s = t0 + (r >> 3);                 // this row's segment
            const bool valid = s < S;
            const int a = valid ? (seg[s] >> 8) : 0;
            // ---- A0: point features of row r (bf16, K padded to 16, constant-1 bias column)
            if (hf == 0) {
                float f[16];
#pragma unroll
                for (int i = 0; i < 8; ++i) { f[i] = fcur[i]; f[8 + i] = 0.0f; }
                store_row16(A0, r, 0, 16, f);
            }
            umma::fence_async_smem();
            umma::fence_before();
            __syncthreads();
            if (tid == 0) {
                if (t0 == 0) umma::bar_wait(bar + 1, wphase);        // weights landed
                umma::fence_after();
                umma::gemm_128xN(tmem, A0, W1, kHid, 16);
                umma::commit(bar);
            }
            fetch(t0 + 16, fcur);                        // next tile's features, in flight meanwhile
            umma::bar_wait(bar, phase);
            phase ^= 1u;
            umma::fence_after();
            // ---- L1 epilogue: (bias already in the GEMM) log2e-scaled ELU -> A1 (bf16),
            //      48 columns per thread
            {
                uint32_t raw[48];
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) umma::tmem_ld16_issue(tmem + lane_base + c0 + 16 * cc, raw + 16 * cc);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    umma::tmem_wait16(raw + 16 * cc);
#ifdef DG_EXP_ELU2
                    uint32_t h[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        h[i] = elu_log2_bf16x2(__uint_as_float(raw[16 * cc + 2 * i]),
                                               __uint_as_float(raw[16 * cc + 2 * i + 1]));
                    const int c = c0 + 16 * cc;
                    *reinterpret_cast<uint4*>(A1 + umma::kmajor_offset(r, c, kHid)) = make_uint4(h[0], h[1], h[2], h[3]);
                    *reinterpret_cast<uint4*>(A1 + umma::kmajor_offset(r, c + 8, kHid)) =
                        make_uint4(h[4], h[5], h[6], h[7]);
#else
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = elu_log2(__uint_as_float(raw[16 * cc + i]));
                    store_row16(A1, r, c0 + 16 * cc, kHid, v);
#endif
                }
            }
            umma::fence_async_smem();
            umma::fence_before();
            __syncthreads();
            if (tid == 0) {
                umma::fence_after();
                umma::gemm_128xN(tmem, A1, W2, kHid, kHid);
                umma::commit(bar);
            }
            umma::bar_wait(bar, phase);
            phase ^= 1u;
            umma::fence_after();
            // ---- L2 epilogue: segment max of the raw accumulator, rounded to bf16
            //      (rounding is monotone: max of rounded == rounded max).  The 8 rows of
            //      a segment are 8 consecutive lanes: a 3-stage transpose-butterfly on
            //      bf16x2 pairs leaves each lane 6 of the 48 columns' maxima.
            uint32_t pk[24];
            {
                // the three 16-column loads in flight together, one wait
                uint32_t raw[48];
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) umma::tmem_ld16_issue(tmem + lane_base + c0 + 16 * cc, raw + 16 * cc);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) umma::tmem_wait16(raw + 16 * cc);
#pragma unroll
                for (int i = 0; i < 24; ++i)
#if DG_L2_NOSEL
                    // rows past the last segment fill whole segments that are never stored
                    pk[i] = umma::pack_bf16(__uint_as_float(raw[2 * i]), __uint_as_float(raw[2 * i + 1]));
#else
                    pk[i] = valid ? umma::pack_bf16(__uint_as_float(raw[2 * i]), __uint_as_float(raw[2 * i + 1]))
                                  : 0xff80ff80u;
#endif
            }
            const bool bA = (lane >> 2) & 1, bB = (lane >> 1) & 1, bC = lane & 1;
            uint32_t qa[12];
#pragma unroll
            for (int j = 0; j < 12; ++j) {
                const uint32_t snd = bA ? pk[j] : pk[12 + j];
                const uint32_t keep = bA ? pk[12 + j] : pk[j];
                qa[j] = bmax2(keep, __shfl_xor_sync(0xffffffffu, snd, 4));
            }
            uint32_t qb[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                const uint32_t snd = bB ? qa[j] : qa[6 + j];
                const uint32_t keep = bB ? qa[6 + j] : qa[j];
                qb[j] = bmax2(keep, __shfl_xor_sync(0xffffffffu, snd, 2));
            }
            uint32_t qc[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const uint32_t snd = bC ? qb[j] : qb[3 + j];
                const uint32_t keep = bC ? qb[3 + j] : qb[j];
                qc[j] = bmax2(keep, __shfl_xor_sync(0xffffffffu, snd, 1));
            }
            if (valid) {
                const int col = c0 + 24 * bA + 12 * bB + 6 * bC;
                uint32_t* dst = acc + a * kAccStride + col;
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    atomicMax(dst + 2 * j, f2o(__uint_as_float(qc[j] << 16)));
                    atomicMax(dst + 2 * j + 1, f2o(__uint_as_float(qc[j] & 0xffff0000u)));
                }
            }
        }
        __syncthreads();
        // ---- pooled embedding = ELU(max + b2), zero when the agent has no valid slot;
        //      two bf16 per thread and store
        uint16_t* out = p.emb + (int64_t(net) * p.n_agents + a0) * kEmb + mod * kHid;
        for (int i = tid; i < na * (kHid / 2); i += kEncThreads) {
            const int a = i / (kHid / 2), c = 2 * (i % (kHid / 2));
            const uint32_t u0 = acc[a * kAccStride + c], u1 = acc[a * kAccStride + c + 1];
            const float v0 = u0 ? elu(o2f(u0) + b2[c]) : 0.0f;
            const float v1 = u1 ? elu(o2f(u1) + b2[c + 1]) : 0.0f;
            *reinterpret_cast<uint32_t*>(out + int64_t(a) * kEmb + c) = umma::pack_bf16(v0, v1);
        }
        if (S == 0 && tid == 0) umma::bar_wait(bar + 1, wphase);   // no tile waited: retire the weight load
        wphase ^= 1u;
        __syncthreads();
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, 128);
}

// ------------------------------------------------------------------ sampling
// Philox4x32-10 (Salmon et al., SC'11): counter (agent, 0, counter lo, counter hi),
// key (seed lo, seed hi) -> four uniforms -> Box-Muller (float64) -> 3 normals.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__device__ __forceinline__ void gaussian3(uint64_t agent, uint64_t seed, uint64_t counter, double* z) {
    uint32_t c[4] = {uint32_t(agent), uint32_t(agent >> 32), uint32_t(counter), uint32_t(counter >> 32)};
    philox4x32_10(c, uint32_t(seed), uint32_t(seed >> 32));
    double u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) u[i] = (double(c[i]) + 0.5) * 2.3283064365386963e-10;   // 2^-32
    const double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
    double s0, c0, s1, c1;
    sincospi(2.0 * u[1], &s0, &c0);
    sincospi(2.0 * u[3], &s1, &c1);
    z[0] = r0 * c0;
    z[1] = r0 * s0;
    z[2] = r1 * c1;
}

// ------------------------------------------------------------------ trunk
constexpr int kTrunkThreads = 256;   // 8 warps: lane quarter = warp % 4, column half = warp / 4
struct TrunkSmem {
    static constexpr int kWe1 = 0;                                  // 64 x 16
    static constexpr int kWe2 = kWe1 + kEgo * 16 * 2;               // 64 x 64
    static constexpr int kWt1 = kWe2 + kEgo * kEgo * 2;             // 128 x 256
    static constexpr int kWt2 = kWt1 + kT1 * 256 * 2;               // 64 x 128
    static constexpr int kAe0 = kWt2 + kT2 * kT1 * 2;               // 128 x 16
    static constexpr int kAe1 = kAe0 + 128 * 16 * 2;                // 128 x 64
    static constexpr int kAt = kAe1 + 128 * kEgo * 2;               // 128 x 256
    static constexpr int kAt2 = kAt + 128 * 256 * 2;                // 128 x 128
    static constexpr int kBias = kAt2 + 128 * kT1 * 2;              // f32: be1 64, be2 64, bt1 128, bt2 64, wh 4x64, bh 4
    static constexpr int kHead = kBias + (64 + 64 + 128 + 64 + 256 + 4) * 4;   // f32 [128][4] partial heads
    static constexpr int kBar = kHead + 128 * 4 * 4;
    static constexpr int kTotal = kBar + 64;
};

#ifndef DG_TRUNK_BATCH
#define DG_TRUNK_BATCH 1
#endif
// NC 16-column TMEM chunks of this thread's row: with DG_TRUNK_BATCH all loads are in
// flight together (one ~70-cycle wait instead of NC), then fn(chunk, v[16]) per chunk
template <int NC, class Fn>
__device__ __forceinline__ void tmem_chunks(uint32_t taddr, Fn&& fn) {
#if DG_TRUNK_BATCH
    uint32_t raw[16 * NC];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) umma::tmem_ld16_issue(taddr + 16 * cc, raw + 16 * cc);
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) umma::tmem_wait16(raw + 16 * cc);
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(raw[16 * cc + i]);
        fn(cc, v);
    }
#else
#pragma unroll 1
    for (int cc = 0; cc < NC; ++cc) {
        float v[16];
        umma::tmem_ld16(taddr + 16 * cc, v);
        fn(cc, v);
    }
#endif
}

__global__ void __launch_bounds__(kTrunkThreads, 1) policy_trunk_kernel(const DgPolicyDesc p) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int net = blockIdx.y + p.first_net;
    const int a0 = blockIdx.x * kTrunkAgents;
    const int q = warp & 3, hf = warp >> 2;
    const int r = 32 * q + lane;                    // tile row = agent a0 + r
    const int agent = a0 + r;
    const bool live = agent < p.n_agents;
    uint8_t* We1 = sm + TrunkSmem::kWe1;
    uint8_t* We2 = sm + TrunkSmem::kWe2;
    uint8_t* Wt1 = sm + TrunkSmem::kWt1;
    uint8_t* Wt2 = sm + TrunkSmem::kWt2;
    uint8_t* Ae0 = sm + TrunkSmem::kAe0;
    uint8_t* Ae1 = sm + TrunkSmem::kAe1;
    uint8_t* At = sm + TrunkSmem::kAt;
    uint8_t* At2 = sm + TrunkSmem::kAt2;
    float* be1 = reinterpret_cast<float*>(sm + TrunkSmem::kBias);
    float* be2 = be1 + 64;
    float* bt1 = be2 + 64;
    float* bt2 = bt1 + 128;
    float* wh = bt2 + 64;
    float* bh = wh + 256;
    float* part = reinterpret_cast<float*>(sm + TrunkSmem::kHead);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + TrunkSmem::kBar);   // [0] mma, [1..3] weights
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + TrunkSmem::kBar + 32);

    const uint8_t* wb = net_base(p, net);
    // the encoder's work queue is drained (stream order): re-arm it for the next forward
    if (p.work_counter && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) p.work_counter[p.first_net] = 0;
    if (warp == 0) umma::tmem_alloc(tmem_slot, 256);
    if (tid == 32) {
        // weights by TMA bulk copies, one mbarrier each, so the ego layers start
        // while the 64 KB trunk matrix is still in flight
        for (int i = 0; i < 4; ++i) umma::bar_init(bar + i, 1);
        expect_tx(bar + 1, kEgo * 16 * 2 + kEgo * kEgo * 2);
        expect_tx(bar + 2, kT1 * 256 * 2);
        expect_tx(bar + 3, kT2 * kT1 * 2);
        bulk_g2s(We1, wb + p.off[DG_POL_W_EGO1], kEgo * 16 * 2, bar + 1);
        bulk_g2s(We2, wb + p.off[DG_POL_W_EGO2], kEgo * kEgo * 2, bar + 1);
        bulk_g2s(Wt1, wb + p.off[DG_POL_W_T1], kT1 * 256 * 2, bar + 2);
        bulk_g2s(Wt2, wb + p.off[DG_POL_W_T2], kT2 * kT1 * 2, bar + 3);
    }
    const int nout = net == 0 ? 3 : 1;
    {
        const float* g;
        g = fsec(p, net, DG_POL_B_EGO1); for (int i = tid; i < 64; i += kTrunkThreads) be1[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_EGO2); for (int i = tid; i < 64; i += kTrunkThreads) be2[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_T1); for (int i = tid; i < 128; i += kTrunkThreads) bt1[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_T2); for (int i = tid; i < 64; i += kTrunkThreads) bt2[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_W_HEAD); for (int i = tid; i < nout * 64; i += kTrunkThreads) wh[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_HEAD); for (int i = tid; i < nout; i += kTrunkThreads) bh[i] = __ldg(g + i);
    }
    // ego features (K padded to 16; warps 0-3) and the pooled road | vehicle embeddings
    // (bf16 rows of 192, 12 of the 24 16-byte chunks per thread)
    if (hf == 0) {
        float f[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = 0.0f;
        if (live) {
            const float* src = p.obs + int64_t(agent) * p.obs_dim;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < p.ego_dim) f[i] = __ldg(src + i);
        }
        store_row16(Ae0, r, 0, 16, f);
    }
    {
        const uint4* e = reinterpret_cast<const uint4*>(p.emb + (int64_t(net) * p.n_agents + agent) * kEmb);
#pragma unroll
        for (int j = 0; j < 12; ++j) {
            const int qq = 12 * hf + j;
            const uint4 v = live ? __ldg(e + qq) : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(At + umma::kmajor_offset(r, kEgo + 8 * qq, 256)) = v;
        }
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    uint32_t phase = 0;

    auto run = [&](uint32_t tcol, const uint8_t* A, const uint8_t* B, int N, int K, int wbar) {
        if (tid == 0) {
            umma::bar_wait(bar + wbar, 0);           // weights landed (TMA)
            umma::fence_after();
            umma::gemm_128xN(tmem + tcol, A, B, N, K);
            umma::commit(bar);
        }
        umma::bar_wait(bar, phase);
        phase ^= 1u;
        umma::fence_after();
    };
    auto sync_for_mma = [&]() {
        umma::fence_async_smem();
        umma::fence_before();
        __syncthreads();
    };

    // ego L1 -> Ae1 (32 columns per thread)
    run(0, Ae0, We1, kEgo, 16, 1);
tmem_chunks<2>(tmem + lane_base + 32 * hf, [&](int cc, float* v) {
        const int c = 32 * hf + 16 * cc;
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = elu(v[i] + be1[c + i]);
        store_row16(Ae1, r, c, kEgo, v);
    });
    sync_for_mma();
    // ego L2 -> At[:, 0:64]
    run(64, Ae1, We2, kEgo, kEgo, 1);
tmem_chunks<2>(tmem + lane_base + 64 + 32 * hf, [&](int cc, float* v) {
        const int c = 32 * hf + 16 * cc;
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = elu(v[i] + be2[c + i]);
        store_row16(At, r, c, 256, v);
    });
    sync_for_mma();
    // trunk L1 -> At2 (64 columns per thread)
    run(128, At, Wt1, kT1, 256, 2);
tmem_chunks<4>(tmem + lane_base + 128 + 64 * hf, [&](int cc, float* v) {
        const int c = 64 * hf + 16 * cc;
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = elu(v[i] + bt1[c + i]);
        store_row16(At2, r, c, kT1, v);
    });
    sync_for_mma();
    // trunk L2 -> registers -> head partial sums over this thread's 32 columns
    run(0, At2, Wt2, kT2, kT1, 3);
    float y[4] = {0.f, 0.f, 0.f, 0.f};
tmem_chunks<2>(tmem + lane_base + 32 * hf, [&](int cc, float* v) {
        const int c = 32 * hf + 16 * cc;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float h = elu(v[i] + bt2[c + i]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < nout) y[j] = fmaf(h, wh[j * 64 + c + i], y[j]);
        }
    });
    if (hf == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) part[4 * r + j] = y[j];
    }
    umma::fence_before();
    __syncthreads();
    if (hf == 0 && live) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < nout) y[j] = bh[j] + (y[j] + part[4 * r + j]);
        if (net == 0) {
            double act[3], lp = 0.0;
            if (p.sample) {
                // a = mu + sigma * eps;  log N(a; mu, sigma) = sum -eps^2/2 - log sigma - log(2 pi)/2
                const float* ls = fsec(p, 0, DG_POL_LOG_STD);
                double z[3];
                gaussian3(uint64_t(agent), p.seed, p.counter, z);
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const double l = double(__ldg(ls + j));
                    act[j] = double(y[j]) + exp(l) * z[j];
                    lp += -0.5 * z[j] * z[j] - l - 0.9189385332046727;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 3; ++j) act[j] = double(y[j]);
            }
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                if (p.mean) p.mean[int64_t(agent) * 3 + j] = y[j];
                if (p.actions) p.actions[int64_t(agent) * 3 + j] = act[j];
                if (p.actions_f32) p.actions_f32[int64_t(agent) * 3 + j] = float(act[j]);
            }
            if (p.log_prob && p.sample) p.log_prob[agent] = float(lp);
        } else if (p.value) {
            p.value[agent] = y[0];
        }
    }
    if (warp == 0) umma::tmem_dealloc(tmem, 256);
}

// ------------------------------------------------------------------ GAE
__global__ void gae_kernel(const double* rewards, const uint8_t* dones, const float* values, int T, int64_t N,
                           double gamma, double lam, float* adv, float* ret) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    double a = 0.0;
    double v_next = double(values[int64_t(T) * N + i]);
    for (int t = T - 1; t >= 0; --t) {
        const int64_t q = int64_t(t) * N + i;
        const double nonterm = dones[q] ? 0.0 : 1.0;
        const double v = double(values[q]);
        const double delta = rewards[q] + gamma * v_next * nonterm - v;
        a = delta + gamma * lam * nonterm * a;
        adv[q] = float(a);
        ret[q] = float(a + v);
        v_next = v;
    }
}

thread_local char g_pol_err[256] = "";

int pol_fail(int code, const char* msg) {
    std::snprintf(g_pol_err, sizeof(g_pol_err), "%s", msg);
    return code;
}

}  // namespace

extern "C" {

const char* dg_policy_last_error(void) { return g_pol_err; }

size_t dg_policy_scratch_bytes(int32_t n_agents, int32_t nets) {
    return size_t(n_agents) * size_t(nets) * kEmb * 2;
}

int dg_policy_forward(const DgPolicyDesc* desc, void* stream) {
    if (!desc || !desc->obs || !desc->weights || !desc->emb) return pol_fail(DG_EINVAL, "dg_policy_forward: null argument");
    const DgPolicyDesc& p = *desc;
    if (p.n_agents < 1) return pol_fail(DG_EINVAL, "dg_policy_forward: n_agents < 1");
    if (p.obs_dim != p.ego_dim + 5 * p.k_road + 7 * p.k_vehicles || p.ego_dim > 16)
        return pol_fail(DG_EINVAL, "dg_policy_forward: observation layout mismatch");
    if (p.k_road > 8 * 255 || p.k_vehicles > 8 * 255) return pol_fail(DG_ENOSUPPORT, "dg_policy_forward: too many slots");
    if (p.first_net != 0 && p.first_net != 1) return pol_fail(DG_EINVAL, "dg_policy_forward: first_net must be 0 or 1");
    const int nets = p.first_net == 1 ? 1 : (p.critic ? 2 : 1);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int kmax = p.k_road > p.k_vehicles ? p.k_road : p.k_vehicles;
    const size_t enc = enc_smem_bytes(kmax);
    // the shared-memory opt-in is per device: remember it per device ordinal
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(policy_encoder_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(policy_trunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     TrunkSmem::kTotal);
        if (e != cudaSuccess) {
            std::snprintf(g_pol_err, sizeof(g_pol_err), "dg_policy_forward: %s", cudaGetErrorString(e));
            return DG_ECUDA;
        }
        if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
    if (enc > 200 * 1024) return pol_fail(DG_ENOSUPPORT, "dg_policy_forward: encoder shared memory too large");
    const int groups = (p.n_agents + kEncAgents - 1) / kEncAgents;
    dim3 g1(groups, nets);
    if (p.work_counter) {
        // persistent: as many CTAs as are resident at once (3 per SM), never more than items
        static int n_sm[64] = {};
        if (dev >= 0 && dev < 64 && n_sm[dev] == 0) cudaDeviceGetAttribute(&n_sm[dev], cudaDevAttrMultiProcessorCount, dev);
        const int sms = dev >= 0 && dev < 64 && n_sm[dev] > 0 ? n_sm[dev] : 148;
        const int items = 2 * nets * groups;
        g1 = dim3(items < DG_ENC_CTAS_PER_SM * sms ? items : DG_ENC_CTAS_PER_SM * sms, 1);
    }
    policy_encoder_kernel<<<g1, kEncThreads, enc, st>>>(p);
    dim3 g2((p.n_agents + kTrunkAgents - 1) / kTrunkAgents, nets);
    policy_trunk_kernel<<<g2, kTrunkThreads, TrunkSmem::kTotal, st>>>(p);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        std::snprintf(g_pol_err, sizeof(g_pol_err), "dg_policy_forward: %s", cudaGetErrorString(err));
        return DG_ECUDA;
    }
    return DG_OK;
}

int dg_gae(const double* rewards, const uint8_t* dones, const float* values, int32_t T, int64_t N, double gamma,
           double lambda, float* advantages, float* returns, void* stream) {
    if (!rewards || !dones || !values || !advantages || !returns) return pol_fail(DG_EINVAL, "dg_gae: null argument");
    if (T < 1 || N < 1) return pol_fail(DG_EINVAL, "dg_gae: need T >= 1 and N >= 1");
    const int threads = 256;
    gae_kernel<<<unsigned((N + threads - 1) / threads), threads, 0, static_cast<cudaStream_t>(stream)>>>(
        rewards, dones, values, T, N, gamma, lambda, advantages, returns);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        std::snprintf(g_pol_err, sizeof(g_pol_err), "dg_gae: %s", cudaGetErrorString(err));
        return DG_ECUDA;
    }
    return DG_OK;
}

}  // extern "C"
