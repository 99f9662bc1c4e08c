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

constexpr int kEncAgents = 64;     // agents per encoder CTA
constexpr int kTrunkAgents = 128;  // agents per trunk CTA (one TMEM lane each)
constexpr int kThreads = 128;
constexpr int kHid = 96;           // road / vehicle encoder width
constexpr int kEgo = 64;
constexpr int kT1 = 128, kT2 = 64;
constexpr int kEmb = 2 * kHid;     // pooled road | vehicle, bf16, per agent and net

__device__ __forceinline__ float elu(float x) { return x > 0.0f ? x : __expf(x) - 1.0f; }

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

__device__ __forceinline__ void copy_to_smem(void* dst, const void* src, int bytes, int tid, int nthreads) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int i = tid; i < bytes / 16; i += nthreads) d[i] = __ldg(s + i);
}

struct PolArgs {
    DgPolicyDesc p;
};

__device__ __forceinline__ const uint8_t* net_base(const DgPolicyDesc& p, int net) {
    return p.weights + int64_t(net) * p.net_stride;
}
__device__ __forceinline__ const float* fsec(const DgPolicyDesc& p, int net, int which) {
    return reinterpret_cast<const float*>(net_base(p, net) + p.off[which]);
}

// ------------------------------------------------------------------ encoder
// Shared memory (bytes): A0 128x16 bf16 | A1 128x96 bf16 | W1 96x16 | W2 96x96 |
// b1 f32[96] | acc u32[64][96] | cnt[64] | segstart[65] | seg u16[64 * 44] | bars
struct EncSmem {
    static constexpr int kA0 = 0;
    static constexpr int kA1 = kA0 + 128 * 16 * 2;
    static constexpr int kW1 = kA1 + 128 * kHid * 2;
    static constexpr int kW2 = kW1 + kHid * 16 * 2;
    static constexpr int kB1 = kW2 + kHid * kHid * 2;
    static constexpr int kAcc = kB1 + kHid * 4;
    static constexpr int kCnt = kAcc + kEncAgents * kHid * 4;
    static constexpr int kSegStart = kCnt + kEncAgents * 4;
    static constexpr int kSeg = kSegStart + (kEncAgents + 4) * 4;
};

__host__ __device__ __forceinline__ int enc_seg_cap(int k_slots) { return kEncAgents * ((k_slots + 7) / 8); }
__host__ __device__ __forceinline__ size_t enc_smem_bytes(int k_max) {
    return size_t(EncSmem::kSeg) + ((size_t(enc_seg_cap(k_max)) * 2 + 15) & ~size_t(15)) + 64;
}

__global__ void __launch_bounds__(kThreads, 2) policy_encoder_kernel(const DgPolicyDesc p) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int net = blockIdx.y;
    const int a0 = blockIdx.x * kEncAgents;
    const int na = min(kEncAgents, p.n_agents - a0);
    uint8_t* A0 = sm + EncSmem::kA0;
    uint8_t* A1 = sm + EncSmem::kA1;
    uint8_t* W1 = sm + EncSmem::kW1;
    uint8_t* W2 = sm + EncSmem::kW2;
    float* b1 = reinterpret_cast<float*>(sm + EncSmem::kB1);
    uint32_t* acc = reinterpret_cast<uint32_t*>(sm + EncSmem::kAcc);
    int* cnt = reinterpret_cast<int*>(sm + EncSmem::kCnt);
    int* segstart = reinterpret_cast<int*>(sm + EncSmem::kSegStart);
    uint16_t* seg = reinterpret_cast<uint16_t*>(sm + EncSmem::kSeg);
    const int kmax = p.k_road > p.k_vehicles ? p.k_road : p.k_vehicles;
    uint8_t* tail = sm + EncSmem::kSeg + ((enc_seg_cap(kmax) * 2 + 15) & ~15);
    uint64_t* bar = reinterpret_cast<uint64_t*>(tail);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tail + 16);

    if (warp == 0) umma::tmem_alloc(tmem_slot, 256);
    if (tid == 0) umma::bar_init(bar, 1);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lane_base = uint32_t(32 * warp) << 16;
    uint32_t phase = 0;
    const uint8_t* wb = net_base(p, net);

    for (int mod = 0; mod < 2; ++mod) {
        const int nf = mod == 0 ? 5 : 7;
        const int kslots = mod == 0 ? p.k_road : p.k_vehicles;
        const int fbase = mod == 0 ? p.ego_dim : p.ego_dim + 5 * p.k_road;
        const int w1 = mod == 0 ? DG_POL_W_ROAD1 : DG_POL_W_VEH1;
        const int w2 = mod == 0 ? DG_POL_W_ROAD2 : DG_POL_W_VEH2;
        const float* gb1 = fsec(p, net, mod == 0 ? DG_POL_B_ROAD1 : DG_POL_B_VEH1);
        const float* gb2 = fsec(p, net, mod == 0 ? DG_POL_B_ROAD2 : DG_POL_B_VEH2);

        // weights of this modality -> shared memory; accumulators cleared
        copy_to_smem(W1, wb + p.off[w1], kHid * 16 * 2, tid, kThreads);
        copy_to_smem(W2, wb + p.off[w2], kHid * kHid * 2, tid, kThreads);
        for (int i = tid; i < kHid; i += kThreads) b1[i] = __ldg(gb1 + i);
        for (int i = tid; i < kEncAgents * kHid; i += kThreads) acc[i] = 0u;

        // valid slot counts: the valid slots are a prefix; warp per agent, 32 slots per probe
        for (int a = warp; a < na; a += kThreads / 32) {
            const float* row = p.obs + int64_t(a0 + a) * p.obs_dim + fbase;
            int c = 0;
            for (int s0 = 0; s0 < kslots; s0 += 32) {
                const int s = s0 + lane;
                bool ok = false;
                if (s < kslots) {
                    const float* f = row + s * nf;
                    ok = mod == 0 ? (__ldg(f + 3) != 0.0f || __ldg(f + 4) != 0.0f) : (__ldg(f + 2) != 0.0f);
                }
                const unsigned b = __ballot_sync(0xffffffffu, ok);
                c += __popc(b);
                if (b != 0xffffffffu) break;
            }
            if (lane == 0) cnt[a] = c;
        }
        __syncthreads();
        if (tid == 0) {
            int s = 0;
            for (int a = 0; a < na; ++a) {
                segstart[a] = s;
                s += (cnt[a] + 7) >> 3;
            }
            segstart[na] = s;
        }
        __syncthreads();
        const int S = segstart[na];
        for (int a = warp; a < na; a += kThreads / 32) {
            const int s0 = segstart[a], n = segstart[a + 1] - s0;
            for (int j = lane; j < n; j += 32) seg[s0 + j] = uint16_t((a << 8) | j);
        }
        umma::fence_async_smem();
        __syncthreads();

        for (int t0 = 0; t0 < S; t0 += 16) {
            // ---- A0: this row's point features (bf16, K padded to 16)
            const int r = tid;
            const int s = t0 + (r >> 3);
            const bool valid = s < S;
            float f[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = 0.0f;
            int a = 0;
            if (valid) {
                const int e = seg[s];
                a = e >> 8;
                int slot = 8 * (e & 255) + (r & 7);
                if (slot >= cnt[a]) slot = 0;                   // duplicate of a valid point
                const float* src = p.obs + int64_t(a0 + a) * p.obs_dim + fbase + slot * nf;
                for (int i = 0; i < nf; ++i) f[i] = __ldg(src + i);
            }
            store_row16(A0, r, 0, 16, f);
            umma::fence_async_smem();
            __syncthreads();
            if (tid == 0) {
                umma::fence_after();
                umma::gemm_128xN(tmem, A0, W1, kHid, 16);
                umma::commit(bar);
            }
            umma::bar_wait(bar, phase);
            phase ^= 1u;
            umma::fence_after();
            // ---- L1 epilogue: +b1, ELU -> A1 (bf16)
#pragma unroll 1
            for (int c = 0; c < kHid; c += 16) {
                float v[16];
                umma::tmem_ld16(tmem + lane_base + c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = elu(v[i] + b1[c + i]);
                store_row16(A1, r, c, kHid, v);
            }
            umma::fence_async_smem();
            umma::fence_before();
            __syncthreads();
            if (tid == 0) {
                umma::fence_after();
                umma::gemm_128xN(tmem + 128, A1, W2, kHid, kHid);
                umma::commit(bar);
            }
            umma::bar_wait(bar, phase);
            phase ^= 1u;
            umma::fence_after();
            // ---- L2 epilogue: segment max of the raw accumulator (8 rows = 8 lanes)
#pragma unroll 1
            for (int c = 0; c < kHid; c += 16) {
                float v[16];
                umma::tmem_ld16(tmem + lane_base + 128 + c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float x = valid ? v[i] : -INFINITY;
                    x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1));
                    x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 2));
                    x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 4));
                    if (valid && (r & 7) == 0) atomicMax(acc + a * kHid + c + i, f2o(x));
                }
            }
            umma::fence_before();
            __syncthreads();
        }
        __syncthreads();
        // ---- pooled embedding = ELU(max + b2), zero when the agent has no valid slot
        uint16_t* out = p.emb + (int64_t(net) * p.n_agents + a0) * kEmb + mod * kHid;
        for (int i = tid; i < na * kHid; i += kThreads) {
            const int a = i / kHid, c = i % kHid;
            const uint32_t u = acc[i];
            const float v = u ? elu(o2f(u) + __ldg(gb2 + c)) : 0.0f;
            const uint32_t pk = umma::pack_bf16(v, 0.0f);
            out[int64_t(a) * kEmb + c] = uint16_t(pk & 0xffffu);
        }
        __syncthreads();
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, 256);
}

// ------------------------------------------------------------------ trunk
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
    static constexpr int kBar = kBias + (64 + 64 + 128 + 64 + 256 + 4) * 4;
    static constexpr int kTotal = kBar + 64;
};

__global__ void __launch_bounds__(kThreads, 1) policy_trunk_kernel(const DgPolicyDesc p) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int net = blockIdx.y;
    const int a0 = blockIdx.x * kTrunkAgents;
    const int r = tid;
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
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + TrunkSmem::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + TrunkSmem::kBar + 16);

    if (warp == 0) umma::tmem_alloc(tmem_slot, 256);
    if (tid == 0) umma::bar_init(bar, 1);
    const uint8_t* wb = net_base(p, net);
    copy_to_smem(We1, wb + p.off[DG_POL_W_EGO1], kEgo * 16 * 2, tid, kThreads);
    copy_to_smem(We2, wb + p.off[DG_POL_W_EGO2], kEgo * kEgo * 2, tid, kThreads);
    copy_to_smem(Wt1, wb + p.off[DG_POL_W_T1], kT1 * 256 * 2, tid, kThreads);
    copy_to_smem(Wt2, wb + p.off[DG_POL_W_T2], kT2 * kT1 * 2, tid, kThreads);
    const int nout = net == 0 ? 3 : 1;
    {
        const float* g;
        g = fsec(p, net, DG_POL_B_EGO1); for (int i = tid; i < 64; i += kThreads) be1[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_EGO2); for (int i = tid; i < 64; i += kThreads) be2[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_T1); for (int i = tid; i < 128; i += kThreads) bt1[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_T2); for (int i = tid; i < 64; i += kThreads) bt2[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_W_HEAD); for (int i = tid; i < nout * 64; i += kThreads) wh[i] = __ldg(g + i);
        g = fsec(p, net, DG_POL_B_HEAD); for (int i = tid; i < nout; i += kThreads) bh[i] = __ldg(g + i);
    }
    // ego features (K padded to 16) and the pooled road | vehicle embeddings
    {
        float f[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = 0.0f;
        if (live) {
            const float* src = p.obs + int64_t(agent) * p.obs_dim;
            for (int i = 0; i < p.ego_dim; ++i) f[i] = __ldg(src + i);
        }
        store_row16(Ae0, r, 0, 16, f);
        const uint4* e = reinterpret_cast<const uint4*>(p.emb + (int64_t(net) * p.n_agents + agent) * kEmb);
#pragma unroll 4
        for (int q = 0; q < kEmb / 8; ++q) {
            const uint4 v = live ? __ldg(e + q) : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(At + umma::kmajor_offset(r, kEgo + 8 * q, 256)) = v;
        }
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lane_base = uint32_t(32 * warp) << 16;
    uint32_t phase = 0;

    auto run = [&](uint32_t tcol, const uint8_t* A, const uint8_t* B, int N, int K) {
        if (tid == 0) {
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

    // ego L1 -> Ae1
    run(0, Ae0, We1, kEgo, 16);
#pragma unroll 1
    for (int c = 0; c < kEgo; c += 16) {
        float v[16];
        umma::tmem_ld16(tmem + lane_base + c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = elu(v[i] + be1[c + i]);
        store_row16(Ae1, r, c, kEgo, v);
    }
    sync_for_mma();
    // ego L2 -> At[:, 0:64]
    run(64, Ae1, We2, kEgo, kEgo);
#pragma unroll 1
    for (int c = 0; c < kEgo; c += 16) {
        float v[16];
        umma::tmem_ld16(tmem + lane_base + 64 + c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = elu(v[i] + be2[c + i]);
        store_row16(At, r, c, 256, v);
    }
    sync_for_mma();
    // trunk L1 -> At2
    run(128, At, Wt1, kT1, 256);
#pragma unroll 1
    for (int c = 0; c < kT1; c += 16) {
        float v[16];
        umma::tmem_ld16(tmem + lane_base + 128 + c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = elu(v[i] + bt1[c + i]);
        store_row16(At2, r, c, kT1, v);
    }
    sync_for_mma();
    // trunk L2 -> registers -> head
    run(0, At2, Wt2, kT2, kT1);
    float y[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < nout; ++j) y[j] = bh[j];
#pragma unroll 1
    for (int c = 0; c < kT2; c += 16) {
        float v[16];
        umma::tmem_ld16(tmem + lane_base + c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float h = elu(v[i] + bt2[c + i]);
            for (int j = 0; j < nout; ++j) y[j] = fmaf(h, wh[j * 64 + c + i], y[j]);
        }
    }
    if (live) {
        if (net == 0) {
            for (int j = 0; j < 3; ++j) {
                if (p.mean) p.mean[int64_t(agent) * 3 + j] = y[j];
                if (p.actions) p.actions[int64_t(agent) * 3 + j] = double(y[j]);
            }
        } else if (p.value) {
            p.value[agent] = y[0];
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, 256);
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
    const int nets = p.critic ? 2 : 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int kmax = p.k_road > p.k_vehicles ? p.k_road : p.k_vehicles;
    const size_t enc = enc_smem_bytes(kmax);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(policy_encoder_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(policy_trunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             TrunkSmem::kTotal);
        attr_set = true;
    }
    if (enc > 200 * 1024) return pol_fail(DG_ENOSUPPORT, "dg_policy_forward: encoder shared memory too large");
    dim3 g1((p.n_agents + kEncAgents - 1) / kEncAgents, nets);
    policy_encoder_kernel<<<g1, kThreads, enc, st>>>(p);
    dim3 g2((p.n_agents + kTrunkAgents - 1) / kTrunkAgents, nets);
    policy_trunk_kernel<<<g2, kThreads, TrunkSmem::kTotal, st>>>(p);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        std::snprintf(g_pol_err, sizeof(g_pol_err), "dg_policy_forward: %s", cudaGetErrorString(err));
        return DG_ECUDA;
    }
    return DG_OK;
}

}  // extern "C"
