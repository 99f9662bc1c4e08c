"""The paper's actor-critic policy MLP on the GPU (BASELINE configs[4]).

The reference package has no policy code; the network is specified only by
the paper (App. E; PPO horizon 128):

* ego encoder      11 -> 64 -> 64           (ELU, ELU)
* road encoder      5 -> 96 -> 96 per point (ELU, ELU), masked max-pool
* vehicle encoder   7 -> 96 -> 96 per slot  (ELU, ELU), masked max-pool
* trunk           256 -> 128 -> 64          (ELU, ELU) on [ego | road | vehicle]
* actor head       64 -> 3 (mean, plus a state-independent log-std)
* critic head      64 -> 1
* separate weights for the actor and the critic.

Padded slots are masked out of the pool (-inf before the max); an agent
with no valid slot gets a zero embedding (the paper leaves that case open).

``PolicyMLP.forward`` runs ``dg_policy_forward`` (csrc/dg_policy.cu): two
tcgen05 kernels reading the step kernel's observation rows where they lie in
HBM.  Weights are random-initialised (torch Linear init, fixed seed) -- there
are no checkpoints offline; ``state_dict`` / ``load_state_dict`` move them.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native as N
from .params import ObsConfig

LAYERS = (  # name, in, out (per net)
    ("ego1", None, 64), ("ego2", 64, 64),
    ("road1", 5, 96), ("road2", 96, 96),
    ("veh1", 7, 96), ("veh2", 96, 96),
    ("t1", 256, 128), ("t2", 128, 64),
)
NETS = ("actor", "critic")
HEAD_OUT = {"actor": 3, "critic": 1}
# padded K of the bf16 tiles (first layers padded to one MMA K step)
TILE_K = {"ego1": 16, "ego2": 64, "road1": 16, "road2": 96, "veh1": 16, "veh2": 96, "t1": 256, "t2": 128}
W_SECTION = {"ego1": "W_EGO1", "ego2": "W_EGO2", "t1": "W_T1", "t2": "W_T2",
             "road1": "W_ROAD1", "road2": "W_ROAD2", "veh1": "W_VEH1", "veh2": "W_VEH2"}
B_SECTION = {"ego1": "B_EGO1", "ego2": "B_EGO2", "road1": "B_ROAD1", "road2": "B_ROAD2",
             "veh1": "B_VEH1", "veh2": "B_VEH2", "t1": "B_T1", "t2": "B_T2"}


def kmajor_tile(w: np.ndarray, K: int) -> np.ndarray:
    """[out][in] weight -> bf16 bytes of the canonical K-major UMMA tile
    (dg_umma.cuh): element (r, k) at ((r/8)*(K/8) + k/8)*128 + (r%8)*16 + (k%8)*2."""
    out, inn = w.shape
    assert out % 8 == 0 and K % 16 == 0 and inn <= K
    full = np.zeros((out, K), dtype=np.float32)
    full[:, :inn] = w
    bf = torch.from_numpy(full).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    r = np.arange(out)[:, None]
    k = np.arange(K)[None, :]
    off = ((r // 8) * (K // 8) + k // 8) * 64 + (r % 8) * 8 + (k % 8)    # in uint16 units
    tile = np.zeros(out * K, dtype=np.uint16)
    tile[off.ravel()] = bf.ravel()
    return tile.view(np.uint8)


LOG2E = float(np.log2(np.e))
LN2 = float(np.log(2.0))


def fold_first_layer(w1: np.ndarray, b1: np.ndarray, K: int = 16) -> np.ndarray:
    """Encoder first layer as the kernel runs it: [W1 | b1] * log2(e) against
    the features with a constant-1 column appended (the bias rides in the
    GEMM; the activation then needs one ex2, dg_policy.cu elu_log2)."""
    out, inn = w1.shape
    assert inn + 1 <= K
    w = np.zeros((out, inn + 1), dtype=np.float64)
    w[:, :inn] = w1
    w[:, inn] = b1
    return (w * LOG2E).astype(np.float32)


def _align16(n: int) -> int:
    return (n + 15) & ~15


class PolicyMLP:
    """Actor-critic weights + the device forward."""

    def __init__(self, obs_config: ObsConfig | None = None, seed: int = 0, device=None,
                 critic: bool = True, head_scale: float = 0.01):
        self.obs_config = obs_config or ObsConfig()
        oc = self.obs_config
        if oc.ego_dim > 16:
            raise ValueError("ego block wider than 16 floats")
        self.critic = bool(critic)
        self.device = torch.device(device if device is not None else "cuda")
        g = torch.Generator().manual_seed(seed)
        self.params = {}
        for net in NETS:
            for name, fin, fout in LAYERS:
                fin = oc.ego_dim if fin is None else fin
                self.params[f"{net}.{name}"] = self._linear(fin, fout, g)
            w, b = self._linear(64, HEAD_OUT[net], g)
            self.params[f"{net}.head"] = (w * head_scale, b * 0.0)
        self.log_std = torch.zeros(3)
        self._blob = None
        self._emb = None
        self._work = torch.zeros(2, dtype=torch.int32, device=self.device)   # encoder work queues (actor, critic)

    @staticmethod
    def _linear(fin, fout, g):
        bound = 1.0 / np.sqrt(fin)                      # torch.nn.Linear default init
        w = (torch.rand((fout, fin), generator=g) * 2 - 1) * bound
        b = (torch.rand((fout,), generator=g) * 2 - 1) * bound
        return w, b

    # ---------------------------------------------------------------- weights
    def state_dict(self) -> dict:
        d = {}
        for k, (w, b) in self.params.items():
            d[k + ".weight"], d[k + ".bias"] = w.clone(), b.clone()
        d["log_std"] = self.log_std.clone()
        return d

    def load_state_dict(self, d: dict) -> None:
        for k in self.params:
            self.params[k] = (d[k + ".weight"].float().cpu(), d[k + ".bias"].float().cpu())
        self.log_std = d.get("log_std", self.log_std).float().cpu()
        self._blob = None

    def _pack(self):
        """One blob per net, sections at the offsets of DgPolicyDesc.off."""
        secs = {}
        for name, _, _ in LAYERS:
            secs[W_SECTION[name]] = lambda net, name=name: kmajor_tile(
                self.params[f"{net}.{name}"][0].numpy(), TILE_K[name])
            secs[B_SECTION[name]] = lambda net, name=name: self.params[f"{net}.{name}"][1].numpy().astype(
                np.float32).view(np.uint8)
        # encoders: bias + log2(e) folded into layer 1, ln 2 into layer 2 (exact algebra)
        for name in ("road", "veh"):
            secs[W_SECTION[name + "1"]] = lambda net, name=name: kmajor_tile(
                fold_first_layer(*(t.numpy() for t in self.params[f"{net}.{name}1"])), 16)
            secs[W_SECTION[name + "2"]] = lambda net, name=name: kmajor_tile(
                (self.params[f"{net}.{name}2"][0].numpy().astype(np.float64) * LN2).astype(np.float32), 96)

        def head_w(net):
            w = np.zeros((4, 64), dtype=np.float32)
            hw = self.params[f"{net}.head"][0].numpy()
            w[:hw.shape[0]] = hw
            return w.view(np.uint8).ravel()

        def head_b(net):
            b = np.zeros(4, dtype=np.float32)
            hb = self.params[f"{net}.head"][1].numpy()
            b[:hb.shape[0]] = hb
            return b.view(np.uint8)

        def log_std(net):
            v = np.zeros(4, dtype=np.float32)
            if net == "actor":
                v[:3] = self.log_std.numpy()
            return v.view(np.uint8)

        secs["W_HEAD"], secs["B_HEAD"], secs["LOG_STD"] = head_w, head_b, log_std
        blobs, offs = [], None
        for net in NETS:
            parts, off, cur = [], [], 0
            for s in N.POL_SECTIONS:
                data = np.ascontiguousarray(secs[s](net)).view(np.uint8).ravel()
                off.append(cur)
                parts.append(data)
                pad = _align16(len(data)) - len(data)
                if pad:
                    parts.append(np.zeros(pad, dtype=np.uint8))
                cur += _align16(len(data))
            blobs.append(np.concatenate(parts))
            offs = offs or off
            assert off == offs
        stride = _align16(max(len(b) for b in blobs))
        blob = np.zeros(stride * len(NETS), dtype=np.uint8)
        for i, b in enumerate(blobs):
            blob[i * stride:i * stride + len(b)] = b
        self._blob = torch.from_numpy(blob).to(self.device)
        self._stride = stride
        self._offs = offs

    # ---------------------------------------------------------------- forward
    def forward(self, obs: torch.Tensor, actions: torch.Tensor | None = None,
                mean: torch.Tensor | None = None, value: torch.Tensor | None = None,
                sample: bool = False, seed: int = 0, counter: int = 0,
                log_prob: torch.Tensor | None = None, actions_f32: torch.Tensor | None = None,
                nets: str = "both", prefix: torch.Tensor | None = None) -> None:
        """Enqueue the forward over every observation row of ``obs``
        ([..., obs_dim] float32, CUDA).  ``actions`` ([..., 3] float64) gets
        the next tick's env input: the actor mean, or with ``sample`` a draw
        mean + exp(log_std) * eps (eps from Philox4x32-10 keyed by ``seed``,
        counter (row, ``counter``)); ``log_prob`` ([...] f32) its log-density,
        ``actions_f32`` ([..., 3]) a float32 copy; ``mean`` ([..., 3] f32),
        ``value`` ([...] f32, needs critic=True).  ``nets``: "both" (default),
        "actor" (no value) or "critic" (value only) -- the two halves can run
        on different streams.  ``prefix`` (int16 [..., 2], the step's
        ``prefix_out`` for these rows) gives the valid road / vehicle slot counts
        so the encoder does not scan the rows for them."""
        if nets not in ("both", "actor", "critic"):
            raise ValueError(f"nets must be 'both', 'actor' or 'critic', not {nets!r}")
        if nets == "actor":
            value = None
        if nets == "critic" and value is None:
            raise ValueError("nets='critic' needs a value output")
        oc = self.obs_config
        if not obs.is_cuda or obs.dtype != torch.float32 or obs.shape[-1] != oc.obs_dim:
            raise ValueError(f"obs must be float32 CUDA [..., {oc.obs_dim}]")
        if not obs.is_contiguous():
            raise ValueError("obs must be contiguous")
        if value is not None and not self.critic:
            raise ValueError("value requested from a policy built with critic=False")
        if self._blob is None:
            self._pack()
        n = obs.numel() // oc.obs_dim
        n_nets = 2 if self.critic else 1
        lib = N.load_library()
        need = int(lib.dg_policy_scratch_bytes(n, n_nets))
        if self._emb is None or self._emb.numel() * 2 < need:
            self._emb = torch.empty(need // 2, dtype=torch.int16, device=self.device)
        d = N.DgPolicyDesc(n_agents=n, obs_dim=oc.obs_dim, ego_dim=oc.ego_dim, k_road=oc.k_road,
                           k_vehicles=oc.k_vehicles, critic=int(self.critic and value is not None),
                           first_net=1 if nets == "critic" else 0,
                           obs=obs.data_ptr(), weights=self._blob.data_ptr(), net_stride=self._stride,
                           emb=self._emb.data_ptr(),
                           mean=mean.data_ptr() if mean is not None else None,
                           actions=actions.data_ptr() if actions is not None else None,
                           value=value.data_ptr() if value is not None else None,
                           sample=int(bool(sample)), seed=int(seed) & (2 ** 64 - 1),
                           counter=int(counter) & (2 ** 64 - 1),
                           log_prob=log_prob.data_ptr() if log_prob is not None else None,
                           actions_f32=actions_f32.data_ptr() if actions_f32 is not None else None,
                           prefix=prefix.data_ptr() if prefix is not None else None,
                           work_counter=self._work.data_ptr())
        for i, o in enumerate(self._offs):
            d.off[i] = o
        for t, dt in ((actions, torch.float64), (mean, torch.float32), (value, torch.float32),
                      (log_prob, torch.float32), (actions_f32, torch.float32)):
            if t is not None and (t.dtype != dt or not t.is_cuda or not t.is_contiguous()):
                raise ValueError("policy outputs must be contiguous CUDA tensors of the documented dtype")
        if prefix is not None and (prefix.dtype != torch.int16 or not prefix.is_cuda or not prefix.is_contiguous()
                                   or prefix.numel() != 2 * n):
            raise ValueError("prefix must be a contiguous int16 CUDA tensor of [..., 2] per observation row")
        st = ct.c_void_p(torch.cuda.current_stream(obs.device).cuda_stream)
        rc = lib.dg_policy_forward(ct.byref(d), st)
        if rc != N.DG_OK:
            raise RuntimeError(f"dg_policy_forward failed ({rc}): {lib.dg_policy_last_error().decode()}")

    def __call__(self, obs: torch.Tensor):
        """(mean [..., 3], value [...]) as new CUDA tensors."""
        lead = obs.shape[:-1]
        mean = torch.empty(lead + (3,), dtype=torch.float32, device=obs.device)
        value = torch.empty(lead, dtype=torch.float32, device=obs.device) if self.critic else None
        self.forward(obs, mean=mean, value=value)
        return mean, value

    def launches(self) -> int:
        return 2


def gae(rewards: torch.Tensor, dones: torch.Tensor, values: torch.Tensor, gamma: float = 0.99,
        lam: float = 0.98):
    """Generalised advantage estimation on the device (``dg_gae``; PPO
    hyper-parameters of PAPER.md:1214-1244 as defaults).  rewards [T][...]
    float64, dones [T][...] (done_t: transition t ended the episode), values
    [T+1][...] float32 with the bootstrap value in row T.  Returns
    (advantages, returns) [T][...] float32."""
    T = rewards.shape[0]
    if tuple(values.shape) != (T + 1,) + tuple(rewards.shape[1:]) or tuple(dones.shape) != tuple(rewards.shape):
        raise ValueError("gae: rewards / dones [T][...], values [T+1][...]")
    r = rewards.to(torch.float64).contiguous()
    d = dones.to(torch.uint8).contiguous()
    v = values.to(torch.float32).contiguous()
    adv = torch.empty(r.shape, dtype=torch.float32, device=r.device)
    ret = torch.empty_like(adv)
    lib = N.load_library()
    st = ct.c_void_p(torch.cuda.current_stream(r.device).cuda_stream)
    rc = lib.dg_gae(r.data_ptr(), d.data_ptr(), v.data_ptr(), T, r[0].numel(), float(gamma), float(lam),
                    adv.data_ptr(), ret.data_ptr(), st)
    if rc != N.DG_OK:
        raise RuntimeError(f"dg_gae failed ({rc}): {lib.dg_policy_last_error().decode()}")
    return adv, ret
