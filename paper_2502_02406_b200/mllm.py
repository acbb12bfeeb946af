"""Toy MLLM stack on B200: LM blocks with cross-attention layers that share ONE
visual-token buffer y, under the STORE_KV / RECOMPUTE_KV activation policies
(reference ``pkg/src/lvxattn/mllm.py``).

Same structure and names as the reference:

  forward   for every block: if it is a CA position, x += flatten(O) W_O with
            (O, L) the distributed cross-attention of project(x, W_Q) against
            project(y, W_K / W_V) (``recompute.ca_forward`` over the LV-XAttn
            ring); then u = x, x = u + tanh(u W1) W2  (mllm.py:274-305).
  backward  reversed blocks: the MLP, then the CA layer with Q re-projected
            from the saved x and, under RECOMPUTE_KV, K/V re-projected from the
            shared y (mllm.py:314-371).  Both policies give the same gradients.

Every LM block is row-local, so the whole stack runs on row shards: rank i
keeps its rows of x (query side) and of y (visual side); the CA layer's ring is
the only cross-row step.  Weight gradients are summed over ranks (all-reduce,
a collective the single-worker reference does not need).

The memory ledger (mllm.py:164-210) counts the bytes this implementation
really keeps: x / y / K / V in the input dtype, the softmax state O, L in the
state dtype (fp32 for bf16 inputs), K/V with ``hkv`` heads.
``measured_activation_bytes`` reads the same categories off the live tensors
(deduplicated by storage, so the shared y counts once); the GPU tests also
hold them against ``torch.cuda.memory_allocated``.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field, replace

import torch
import torch.distributed as dist

from .comm import DeviceContext
from .kernels import default_scale, state_dtype
from .recompute import (ActivationPolicy, CrossAttentionGrads, CrossAttentionWeights, OpCounter,
                        SavedCA, VisualGradSink, ca_backward, ca_forward)
from .strategies import ShardSpec

_DTYPES = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}


def dtype_from_name(name: str) -> torch.dtype:
    try:
        return _DTYPES[name]
    except KeyError:
        raise ValueError(f"unknown dtype {name!r}; expected one of {sorted(_DTYPES)}")


@dataclass(frozen=True)
class ToyMllmConfig:
    """mllm.py:40-111 (+ ``hkv`` for GQA; None = h, the reference's MHA)."""

    num_lm_blocks: int
    ca_positions: tuple
    d_embed: int
    h: int
    d: int
    frames: int
    tokens_per_frame: int
    s_q: int
    dtype: str = "bf16"
    hkv: int | None = None

    def __post_init__(self):
        object.__setattr__(self, "ca_positions", tuple(self.ca_positions))
        if self.num_lm_blocks < 0:
            raise ValueError(f"num_lm_blocks must be >= 0, got {self.num_lm_blocks}")
        for name in ("d_embed", "h", "d", "tokens_per_frame", "s_q"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.frames < 0:
            raise ValueError(f"frames must be >= 0, got {self.frames}")
        if len(set(self.ca_positions)) != len(self.ca_positions):
            raise ValueError(f"duplicate ca_positions: {self.ca_positions}")
        for p in self.ca_positions:
            if not 0 <= p < self.num_lm_blocks:
                raise ValueError(f"ca_position {p} out of range [0, {self.num_lm_blocks})")
        if self.hkv is not None and (self.hkv < 1 or self.h % self.hkv):
            raise ValueError(f"hkv {self.hkv} must divide h {self.h}")
        dtype_from_name(self.dtype)

    @property
    def kv_heads(self) -> int:
        return self.h if self.hkv is None else self.hkv

    @property
    def s_kv(self) -> int:
        return self.frames * self.tokens_per_frame

    @property
    def num_ca_layers(self) -> int:
        return len(self.ca_positions)

    @property
    def torch_dtype(self) -> torch.dtype:
        return dtype_from_name(self.dtype)

    @property
    def elem_bytes(self) -> int:
        return torch.empty((), dtype=self.torch_dtype).element_size()

    @property
    def state_bytes(self) -> int:
        return torch.empty((), dtype=state_dtype(self.torch_dtype)).element_size()

    @classmethod
    def from_dict(cls, data: dict) -> "ToyMllmConfig":
        fields = {"num_lm_blocks", "ca_positions", "d_embed", "h", "d", "frames",
                  "tokens_per_frame", "s_q", "dtype", "hkv"}
        unknown = set(data) - fields
        if unknown:
            raise ValueError(f"unknown config fields: {sorted(unknown)}")
        missing = fields - set(data) - {"dtype", "hkv"}
        if missing:
            raise ValueError(f"missing config fields: {sorted(missing)}")
        return cls(**data)

    @classmethod
    def from_json(cls, text: str) -> "ToyMllmConfig":
        return cls.from_dict(json.loads(text))

    def as_dict(self) -> dict:
        out = {"num_lm_blocks": self.num_lm_blocks, "ca_positions": list(self.ca_positions),
               "d_embed": self.d_embed, "h": self.h, "d": self.d, "frames": self.frames,
               "tokens_per_frame": self.tokens_per_frame, "s_q": self.s_q, "dtype": self.dtype}
        if self.hkv is not None:
            out["hkv"] = self.hkv
        return out


# the reference's shipped preset (mllm.py:110-111) in bf16
TOY_CONFIG = ToyMllmConfig(num_lm_blocks=8, ca_positions=(1, 3, 5, 7), d_embed=128, h=2, d=64,
                           frames=16, tokens_per_frame=729, s_q=64, dtype="bf16")


@dataclass
class ModelParams:
    """CA weights per position (``recompute.CrossAttentionWeights``) and LM
    block weights [(w1, w2)], all on the device (mllm.py:114-161)."""

    ca: dict
    lm: list

    @classmethod
    def init_random(cls, config: ToyMllmConfig, seed: int = 0,
                    device: torch.device | str = "cuda") -> "ModelParams":
        """U[-0.5/sqrt(e), 0.5/sqrt(e)] weights (mllm.py:136-152), device RNG."""
        e, hd, hkd = config.d_embed, config.h * config.d, config.kv_heads * config.d
        dt = config.torch_dtype
        gen = torch.Generator(device=device).manual_seed(seed)
        sc = 0.5 / e ** 0.5

        def u(*shape):
            return ((torch.rand(*shape, device=device, generator=gen, dtype=torch.float64) * 2
                     - 1) * sc).to(dt)
        ca = {p: CrossAttentionWeights(u(e, hd), u(e, hkd), u(e, hkd), u(hd, e), config.h,
                                       config.kv_heads) for p in config.ca_positions}
        lm = [(u(e, e), u(e, e)) for _ in range(config.num_lm_blocks)]
        return cls(ca=ca, lm=lm)

    def total_bytes(self) -> int:
        n = 0
        for w in self.ca.values():
            n += sum(t.numel() * t.element_size() for t in (w.w_q, w.w_k, w.w_v, w.w_o))
        for w1, w2 in self.lm:
            n += (w1.numel() + w2.numel()) * w1.element_size()
        return n


@dataclass(frozen=True)
class MemoryLedger:
    """mllm.py:164-187: what a policy keeps alive through the forward pass."""

    params_bytes: int
    visual_features_y: int
    per_layer_saved_x: int
    per_layer_saved_o_l: int
    per_layer_saved_kv: int
    num_ca_layers: int
    peak_total: int

    def as_dict(self) -> dict:
        return {"params_bytes": self.params_bytes, "visual_features_y": self.visual_features_y,
                "per_layer_saved_x": self.per_layer_saved_x,
                "per_layer_saved_o_l": self.per_layer_saved_o_l,
                "per_layer_saved_kv": self.per_layer_saved_kv,
                "num_ca_layers": self.num_ca_layers, "peak_total": self.peak_total}


def analytic_ledger(config: ToyMllmConfig, policy: ActivationPolicy, n: int = 1,
                    rank: int = 0) -> MemoryLedger:
    """mllm.py:190-210 for this implementation's layout, per rank of an n-way
    row sharding (n = 1: the whole model): x, y, K, V in the input dtype; O, L
    in the state dtype; K/V with hkv heads; parameters replicated."""
    policy = ActivationPolicy(policy)
    b, bs = config.elem_bytes, config.state_bytes
    e, h, hkv, d = config.d_embed, config.h, config.kv_heads, config.d
    c = config.num_ca_layers
    shards = ShardSpec.balanced(config.s_q, config.s_kv, n)
    sq, skv = shards.q_sizes[rank], shards.kv_sizes[rank]
    params = (c * (2 * e * h * d + 2 * e * hkv * d) + config.num_lm_blocks * 2 * e * e) * b
    y = skv * e * b
    x = sq * e * b if c else 0
    o_l = (sq * h * d + sq * h) * bs if c else 0
    kv = 2 * skv * hkv * d * b if (c and policy is ActivationPolicy.STORE_KV) else 0
    peak = params + y + c * (x + o_l + kv)   # nothing is freed before the backward
    return MemoryLedger(params, y, x, o_l, kv, c, peak)


def max_frames_under_budget(config: ToyMllmConfig, policy: ActivationPolicy, budget_bytes: int,
                            n: int = 1) -> int:
    """mllm.py:374-397: largest frame count whose analytic peak (per rank of an
    n-way sharding, rank 0 holds the largest shard) fits the budget."""
    if budget_bytes <= 0:
        raise ValueError(f"budget must be positive, got {budget_bytes}")

    def fits(frames: int) -> bool:
        return analytic_ledger(replace(config, frames=frames), policy, n).peak_total <= \
            budget_bytes

    if not fits(0):
        return 0
    if fits(1 << 60):
        raise ValueError("budget admits an absurd frame count; check inputs")
    # the peak grows with the frame count: set the answer's bits high to low
    frames = 0
    for bit in range(59, -1, -1):
        if fits(frames | (1 << bit)):
            frames |= 1 << bit
    return frames


@dataclass
class SavedActivations:
    policy: ActivationPolicy
    y: torch.Tensor
    lm_inputs: list = field(default_factory=list)
    ca: dict = field(default_factory=dict)     # position -> recompute.SavedCA


def measured_activation_bytes(saved: SavedActivations) -> dict:
    """mllm.py:220-240 on live device tensors, deduplicated by storage."""
    seen: set = set()

    def count(t) -> int:
        if t is None:
            return 0
        key = (t.untyped_storage().data_ptr(), t.storage_offset(), t.numel())
        if key in seen:
            return 0
        seen.add(key)
        return t.numel() * t.element_size()

    out = {"visual_features_y": count(saved.y), "saved_x": 0, "saved_o_l": 0, "saved_kv": 0}
    for s in saved.ca.values():
        out["saved_x"] += count(s.x)
        out["saved_o_l"] += count(s.state.O) + count(s.state.L)
        if s.kv is not None:
            out["saved_kv"] += count(s.kv[0]) + count(s.kv[1])
    return out


@dataclass
class MllmGradients:
    d_x0: torch.Tensor
    d_y: torch.Tensor
    ca: dict      # position -> recompute.CrossAttentionGrads
    lm: list      # [(g_w1, g_w2)]


def _ctx_shards(config: ToyMllmConfig, ctx: DeviceContext | None):
    ctx = ctx if ctx is not None else DeviceContext(0, 1)
    return ctx, ShardSpec.balanced(config.s_q, config.s_kv, ctx.n)


def mllm_forward(x0: torch.Tensor, y: torch.Tensor, params: ModelParams,
                 config: ToyMllmConfig, policy: ActivationPolicy,
                 ctx: DeviceContext | None = None):
    """Run the block stack on this rank's rows (x0 [sq_i, e], y [skv_i, e]);
    returns (output, saved activations, ledger) like mllm.py:274-305."""
    policy = ActivationPolicy(policy)
    ctx, shards = _ctx_shards(config, ctx)
    sq, skv = shards.q_sizes[ctx.rank], shards.kv_sizes[ctx.rank]
    if tuple(x0.shape) != (sq, config.d_embed):
        raise ValueError(f"x0 shape {tuple(x0.shape)} != ({sq}, {config.d_embed})")
    if tuple(y.shape) != (skv, config.d_embed):
        raise ValueError(f"y shape {tuple(y.shape)} != ({skv}, {config.d_embed})")
    scale = default_scale(config.d)
    ca_set = set(config.ca_positions)
    saved = SavedActivations(policy=policy, y=y)
    x = x0
    for blk in range(config.num_lm_blocks):
        if blk in ca_set:
            x, saved.ca[blk] = ca_forward(ctx, shards, x, y, params.ca[blk], policy, scale)
        saved.lm_inputs.append(x)
        w1, w2 = params.lm[blk]
        x = x + torch.tanh(x @ w1) @ w2
    return x, saved, analytic_ledger(config, policy, ctx.n, ctx.rank)


def mllm_backward(d_out: torch.Tensor, saved: SavedActivations, y: torch.Tensor,
                  params: ModelParams, config: ToyMllmConfig, policy: ActivationPolicy,
                  counter: OpCounter | None = None,
                  ctx: DeviceContext | None = None) -> MllmGradients:
    """mllm.py:314-371; weight gradients are all-reduced when n > 1."""
    policy = ActivationPolicy(policy)
    if saved.policy is not policy:
        raise ValueError(f"saved activations were produced under policy "
                         f"{saved.policy.value!r}, not {policy.value!r}")
    ctx, shards = _ctx_shards(config, ctx)
    scale = default_scale(config.d)
    ca_set = set(config.ca_positions)
    g = d_out
    # the visual tokens' gradient sums over the CA layers (mllm.py:368): each
    # layer leaves its [dK | dV] in the sink; one GEMM over all layers at the end
    ca_order = [b for b in reversed(range(config.num_lm_blocks)) if b in ca_set]
    sink = VisualGradSink(y, [params.ca[b].kv_weight().shape[1] for b in ca_order])
    ca_grads: dict = {}
    lm_grads: list = [None] * config.num_lm_blocks
    for blk in reversed(range(config.num_lm_blocks)):
        w1, w2 = params.lm[blk]
        u = saved.lm_inputs[blk]
        t = torch.tanh(u @ w1)
        d_pre = (g @ w2.T) * (1.0 - t * t)
        gw1, gw2 = u.T @ d_pre, t.T @ g
        if ctx.n > 1:
            for tt in (gw1, gw2):
                dist.all_reduce(tt, group=ctx.group)
        lm_grads[blk] = (gw1, gw2)
        g = g + d_pre @ w1.T
        if blk in ca_set:
            if blk not in saved.ca:
                raise ValueError(f"layer {blk}: missing saved activations")
            gr: CrossAttentionGrads = ca_backward(ctx, shards, g, saved.ca[blk], y,
                                                  params.ca[blk], scale, counter=counter,
                                                  dy_sink=sink)
            ca_grads[blk] = gr
            g = gr.d_x
    d_y = sink.finish(ctx, dtype=y.dtype)
    return MllmGradients(d_x0=g, d_y=d_y, ca=ca_grads, lm=lm_grads)


def live_activation_bytes(saved: SavedActivations) -> int:
    """Everything ``saved`` keeps alive (ledger categories + the LM inputs)."""
    m = measured_activation_bytes(saved)
    lm = sum(t.numel() * t.element_size() for t in saved.lm_inputs)
    return sum(m.values()) + lm


__all__ = ["ToyMllmConfig", "TOY_CONFIG", "ModelParams", "MemoryLedger", "analytic_ledger",
           "max_frames_under_budget", "SavedActivations", "measured_activation_bytes",
           "MllmGradients", "mllm_forward", "mllm_backward", "live_activation_bytes",
           "ActivationPolicy", "OpCounter", "SavedCA"]
