"""A stack of MoE layers (config c4's "block stack ... with fused small-message
comm"): L MoELayers applied in sequence, backward in reverse, with the
replicated gate gradients of all layers reduced over the EP group through
gradient-bucket fusion (moe_grad_buckets, the reference's make_gradient_buckets
+ GradBucket, collectives.cpp:120-162) instead of one all-reduce per layer.

Each layer is built with gate_grad_reduce="caller"; after a layer's backward
its (dwg, dbg) ids are pushed in arrival order (back to front), and a bucket
flushes -- pack, ONE ncclAllReduce, unpack on the stream -- when its last
gradient arrives, so with the default capacity (two layers per bucket) the
fused all-reduce of the upper layers overlaps the backward of the lower ones.
Attention / dense sublayers of a GPT block are out of scope.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Tuple

import torch

from .layer import EPGroup, MoEConfig, MoELayer
from .moesim import GradBuckets

_GOLD = 0x9E3779B97F4A7C15


class MoEStack:
    def __init__(self, cfg: MoEConfig, num_layers: int, ep: Optional[EPGroup] = None, device=None,
                 layers_per_bucket: int = 2):
        if num_layers < 1:
            from ._lib import ConfigError
            raise ConfigError("stack.num_layers: must be >= 1")
        lcfg = dataclasses.replace(cfg, gate_grad_reduce="caller" if ep is not None else "layer")
        self.cfg, self.ep = lcfg, ep
        self.layers: List[MoELayer] = [MoELayer(lcfg, ep=ep, device=device)
                                       for _ in range(num_layers)]
        self.buckets = None
        self._per_bucket = max(1, layers_per_bucket)

    # the stack mirrors MoELayer's surface where the bench / tests use it
    @property
    def capacity(self) -> int:
        return self.layers[0].capacity

    def init_params(self, seed: int, gate_bias: Optional[torch.Tensor] = None) -> None:
        for i, layer in enumerate(self.layers):
            layer.init_params((seed ^ (_GOLD * (i + 1))) & ((1 << 64) - 1), gate_bias=gate_bias)
        if self.ep is not None and self.buckets is None:
            # the gradient tensors exist once the parameters do
            grads, ids = [], []
            for i, layer in enumerate(self.layers):
                grads += [layer.grads["dwg"], layer.grads["dbg"]]
                ids += [2 * i, 2 * i + 1]
            self.buckets = GradBuckets(ids, capacity=2 * self._per_bucket, grads=grads,
                                       ep=self.ep, scale=1.0)

    def make_input(self, seed: int, tensor_id: int = 6) -> torch.Tensor:
        return self.layers[0].make_input(seed, tensor_id)

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        for layer in self.layers:
            x = layer.forward(x, stream=stream)
        return x

    def backward(self, dy: torch.Tensor, d_aux: float = 0.0, stream=None) -> torch.Tensor:
        if self.buckets is not None:
            self.buckets.reset()
        for i in range(len(self.layers) - 1, -1, -1):
            dy = self.layers[i].backward(dy, d_aux=d_aux, stream=stream)
            if self.buckets is not None:
                self.buckets.push(2 * i, stream=stream)
                self.buckets.push(2 * i + 1, stream=stream)
        return dy

    def set_profiling(self, on: bool) -> None:
        for layer in self.layers:
            layer.set_profiling(on)

    def phase_list(self, which: Optional[str] = None) -> List[Tuple[str, float]]:
        """Phases of the last call (or forward / backward) of every layer."""
        out = []
        for layer in self.layers:
            out += layer.phase_list(which)
        return out

    def phase_times(self) -> Dict[str, float]:
        out: Dict[str, float] = {}
        for name, ms in self.phase_list():
            out[name] = out.get(name, 0.0) + ms
        return out

    def close(self) -> None:
        if self.buckets is not None:
            self.buckets.close()
            self.buckets = None
        for layer in self.layers:
            layer.close()
