"""Ring-of-sections inference (K7) over moe_ring_* (include/moe_b200.h).

N MoE layers whose expert sections sit in pinned host memory rotate through
K HBM slots in the reference's calculation-release-load order
(ring_offload.cpp:31-50); the returned timeline carries the metrics the
reference's infer-sim mode reports (report.cpp:172-187).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional

import torch

from ._lib import RingDesc, RingTimeline, call, lib
from .layer import MoELayer, T_B1, T_B2, T_W1, T_W2, fill_uniform, substream_seed, _stream


class RingOfSections:
    def __init__(self, layer: MoELayer, num_layers: int, ring_slots: int, seed: int = 0,
                 gate_weights: Optional[List[torch.Tensor]] = None):
        import math
        self.layer = layer
        self.N, self.K = num_layers, ring_slots
        c = layer.cfg
        self.section_bytes = int(lib.moe_ring_section_bytes(layer._h))
        self.host = []
        self.gates = []
        bd, bf = 1.0 / math.sqrt(c.d_model), 1.0 / math.sqrt(c.d_ff)
        El = layer.El
        for i in range(num_layers):
            # per-layer expert weights generated on the device then packed into pinned host memory
            w1 = torch.empty(El, c.d_ff, c.d_model, dtype=c.dtype, device=layer.device)
            b1 = torch.empty(El, c.d_ff, dtype=torch.float32, device=layer.device)
            w2 = torch.empty(El, c.d_model, c.d_ff, dtype=c.dtype, device=layer.device)
            b2 = torch.empty(El, c.d_model, dtype=torch.float32, device=layer.device)
            for j in range(El):
                e = layer.rank * El + j
                s = substream_seed(seed, 100 + i, e)
                fill_uniform(w1[j], substream_seed(s, T_W1, 0), -bd, bd)
                fill_uniform(b1[j], substream_seed(s, T_B1, 0), -bd, bd)
                fill_uniform(w2[j], substream_seed(s, T_W2, 0), -bf, bf)
                fill_uniform(b2[j], substream_seed(s, T_B2, 0), -bf, bf)
            torch.cuda.synchronize()
            h = torch.empty(self.section_bytes, dtype=torch.uint8, pin_memory=True)
            call("moe_ring_pack_section", layer._h, w1.data_ptr(), b1.data_ptr(), w2.data_ptr(),
                 b2.data_ptr(), h.data_ptr())
            self.host.append(h)
            del w1, b1, w2, b2
            if gate_weights is not None:
                self.gates.append(gate_weights[i])
            else:
                wg = torch.empty(c.num_experts, c.d_model, dtype=c.dtype, device=layer.device)
                fill_uniform(wg, substream_seed(seed, 200 + i, 0), -bd, bd)
                self.gates.append(wg)
        self._hp = (C.c_void_p * num_layers)(*[h.data_ptr() for h in self.host])
        self._gp = (C.c_void_p * num_layers)(*[g.data_ptr() for g in self.gates])
        desc = RingDesc(num_layers, ring_slots, C.cast(self._hp, C.c_void_p),
                        C.cast(self._gp, C.c_void_p), None)
        h = C.c_void_p()
        call("moe_ring_create", layer._h, C.byref(desc), C.byref(h))
        self._h = h

    def section_tensors(self, i: int) -> Dict[str, torch.Tensor]:
        """Device copies of layer i's expert weights (for reference checks)."""
        c, El = self.layer.cfg, self.layer.El
        raw = self.host[i].cuda()
        es = 2 if c.dtype == torch.bfloat16 else 4
        al = lambda v: (v + 255) // 256 * 256  # noqa: E731
        o_b1 = al(El * c.d_ff * c.d_model * es)
        o_w2 = al(o_b1 + El * c.d_ff * 4)
        o_b2 = al(o_w2 + El * c.d_model * c.d_ff * es)
        w1 = raw[: El * c.d_ff * c.d_model * es].view(c.dtype).view(El, c.d_ff, c.d_model)
        b1 = raw[o_b1:o_b1 + El * c.d_ff * 4].view(torch.float32).view(El, c.d_ff)
        w2 = raw[o_w2:o_w2 + El * c.d_model * c.d_ff * es].view(c.dtype).view(El, c.d_model, c.d_ff)
        b2 = raw[o_b2:o_b2 + El * c.d_model * 4].view(torch.float32).view(El, c.d_model)
        return {"wg": self.gates[i], "w1": w1, "b1": b1, "w2": w2, "b2": b2}

    def run(self, x: torch.Tensor, stream=None):
        y = torch.empty_like(x)
        arrs = [(C.c_float * self.N)() for _ in range(4)]
        tl = RingTimeline()
        tl.load_start, tl.load_end, tl.compute_start, tl.compute_end = [
            C.cast(a, C.c_void_p) for a in arrs]
        call("moe_ring_run", self._h, x.data_ptr(), y.data_ptr(), C.byref(tl), _stream(stream))
        timeline = {
            "load_start": list(arrs[0]), "load_end": list(arrs[1]),
            "compute_start": list(arrs[2]), "compute_end": list(arrs[3]),
            "makespan_ms": tl.makespan_ms, "compute_total_ms": tl.compute_total_ms,
            "peak_gpu_bytes": tl.peak_gpu_bytes, "baseline_gpu_bytes": tl.baseline_gpu_bytes,
            "slots": tl.slots, "clamped": bool(tl.clamped), "section_bytes": self.section_bytes,
        }
        return y, timeline

    def close(self):
        if getattr(self, "_h", None):
            call("moe_ring_destroy", self._h)
            self._h = None
