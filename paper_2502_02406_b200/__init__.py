"""B200-native LV-XAttn: distributed cross-attention for very long visual
contexts (arXiv 2502.02406), drop-in for the reference package ``lvxattn``'s
hot path (kernels + query/KV-rotation strategies).

Kernels: hand-written sm_100a CUDA (tcgen05/TMEM/TMA) in ``liblvx_b200.so``
behind the C ABI of ``include/lvx_b200.h``.  Schedulers (``strategies``): one
rank per GPU, or thread ranks sharing one GPU; the ring hops are copy-engine
transfers into the peers' arenas (``comm``).  There is no CPU fallback.

Submodules beyond the kernels and schedulers: ``recompute`` (the CA layer with
the K/V recompute), ``mllm`` (the toy MLLM stack, memory ledger, frame
budget), ``host_pipeline`` (host-resident inputs streamed over PCIe),
``analytics`` (the cost model), ``volumes`` (byte closed forms),
``tensorio`` (LVXT files, file-to-file runs).
"""
from .comm import (ClusterError, ClusterSpec, CollectiveTimeout, DeviceContext, Instant,
                   TransportStats, WorkerFailed)
from .kernels import (AttentionState, GradientBundle, attention_row_stats, blockwise_attention,
                      blockwise_attention_backward, default_scale, dense_attention,
                      dense_attention_backward, empty_state, merge_states, project,
                      project_backward, validate_qkv)
from .strategies import (RoundRecord, RoundTrace, RunResult, ShardSpec, StepGraph, StrategyKind,
                         head_parallel_backward, head_parallel_forward,
                         lvx_backward, lvx_forward, partition_rows, ring_backward,
                         ring_backward_reference_schedule, ring_forward,
                         run_distributed, run_rank)
from . import analytics, tensorio, volumes

__version__ = "0.1.0"

__all__ = [
    "AttentionState", "ClusterError", "ClusterSpec", "CollectiveTimeout", "DeviceContext",
    "GradientBundle", "Instant", "RoundRecord", "RoundTrace", "RunResult", "ShardSpec",
    "StepGraph", "StrategyKind", "TransportStats", "WorkerFailed", "attention_row_stats",
    "blockwise_attention", "blockwise_attention_backward", "default_scale", "dense_attention",
    "dense_attention_backward", "empty_state", "lvx_backward", "lvx_forward", "merge_states",
    "partition_rows", "project", "project_backward", "ring_backward",
    "ring_backward_reference_schedule", "ring_forward",
    "run_distributed", "run_rank", "validate_qkv", "volumes", "analytics", "tensorio",
]
