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


def make_sections(layer: MoELayer, num_layers: int, seed: int,
                  gate_weights: Optional[List[torch.Tensor]] = None):
    """Per-layer expert sections (SplitMix64 substreams 100+i) packed into
    pinned host memory, and the resident gate weights (substreams 200+i)."""
    import math
    c = layer.cfg
    section_bytes = int(lib.moe_ring_section_bytes(layer._h))
    host, gates = [], []
    bd, bf = 1.0 / math.sqrt(c.d_model), 1.0 / math.sqrt(c.d_ff)
    El = layer.El
    for i in range(num_layers):
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
        h = torch.empty(section_bytes, dtype=torch.uint8, pin_memory=True)
        call("moe_ring_pack_section", layer._h, w1.data_ptr(), b1.data_ptr(), w2.data_ptr(),
             b2.data_ptr(), h.data_ptr())
        host.append(h)
        del w1, b1, w2, b2
        if gate_weights is not None:
            gates.append(gate_weights[i])
        else:
            wg = torch.empty(c.num_experts, c.d_model, dtype=c.dtype, device=layer.device)
            fill_uniform(wg, substream_seed(seed, 200 + i, 0), -bd, bd)
            gates.append(wg)
    return section_bytes, host, gates


def section_tensors(layer: MoELayer, host: torch.Tensor, gate: torch.Tensor) -> Dict[str, torch.Tensor]:
    """Device copies of one packed section's expert weights (for reference checks)."""
    c, El = layer.cfg, layer.El
    raw = host.cuda()
    es = 2 if c.dtype == torch.bfloat16 else 4
    al = lambda v: (v + 255) // 256 * 256  # noqa: E731
    o_b1 = al(El * c.d_ff * c.d_model * es)
    o_w2 = al(o_b1 + El * c.d_ff * 4)
    o_b2 = al(o_w2 + El * c.d_model * c.d_ff * es)
    w1 = raw[: El * c.d_ff * c.d_model * es].view(c.dtype).view(El, c.d_ff, c.d_model)
    b1 = raw[o_b1:o_b1 + El * c.d_ff * 4].view(torch.float32).view(El, c.d_ff)
    w2 = raw[o_w2:o_w2 + El * c.d_model * c.d_ff * es].view(c.dtype).view(El, c.d_model, c.d_ff)
    b2 = raw[o_b2:o_b2 + El * c.d_model * 4].view(torch.float32).view(El, c.d_model)
    return {"wg": gate, "w1": w1, "b1": b1, "w2": w2, "b2": b2}


class RingOfSections:
    def __init__(self, layer: MoELayer, num_layers: int, ring_slots: int, seed: int = 0,
                 gate_weights: Optional[List[torch.Tensor]] = None):
        self.layer = layer
        self.N, self.K = num_layers, ring_slots
        self.section_bytes, self.host, self.gates = make_sections(layer, num_layers, seed,
                                                                  gate_weights)
        self._hp = (C.c_void_p * num_layers)(*[h.data_ptr() for h in self.host])
        self._gp = (C.c_void_p * num_layers)(*[g.data_ptr() for g in self.gates])
        desc = RingDesc(num_layers, ring_slots, C.cast(self._hp, C.c_void_p),
                        C.cast(self._gp, C.c_void_p), None)
        h = C.c_void_p()
        call("moe_ring_create", layer._h, C.byref(desc), C.byref(h))
        self._h = h

    def section_tensors(self, i: int) -> Dict[str, torch.Tensor]:
        """Device copies of layer i's expert weights (for reference checks)."""
        return section_tensors(self.layer, self.host[i], self.gates[i])

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


class Prefetch2D:
    """2D prefetch with the Algorithm-1 CPU cache (moe_prefetch_*, SURVEY.md §8
    f3): N layers' expert sections in a backing-store file, pinned CPU blocks
    managed by SparseCache, lookahead + 1 HBM slots.  run(x, steps) returns y,
    per-(step, layer) records (cache outcome, backing-store I/O time, H2D and
    compute timeline) and a summary (makespan, stall, bytes)."""

    def __init__(self, layer: MoELayer, num_layers: int, lookahead: int, cpu_size: int,
                 backing_path: str, threshold: float = 1.0, beta: float = 1.0,
                 decay_steps: int = 1, flush_period: int = 0, seed: int = 0,
                 gate_weights: Optional[List[torch.Tensor]] = None):
        from ._lib import CacheParams, PrefetchDesc
        self.layer = layer
        self.N = num_layers
        self.section_bytes, self.host, self.gates = make_sections(layer, num_layers, seed,
                                                                  gate_weights)
        self._hp = (C.c_void_p * num_layers)(*[h.data_ptr() for h in self.host])
        self._gp = (C.c_void_p * num_layers)(*[g.data_ptr() for g in self.gates])
        self._path = backing_path.encode()
        desc = PrefetchDesc(num_layers, lookahead,
                            CacheParams(cpu_size, float(threshold), float(beta), decay_steps),
                            flush_period, C.cast(self._hp, C.c_void_p),
                            C.cast(self._gp, C.c_void_p), self._path)
        h = C.c_void_p()
        call("moe_prefetch_create", layer._h, C.byref(desc), C.byref(h))
        self._h = h

    def section_tensors(self, i: int) -> Dict[str, torch.Tensor]:
        return section_tensors(self.layer, self.host[i], self.gates[i])

    def run(self, x: torch.Tensor, steps: int, stream=None):
        from ._lib import PrefetchRecord, PrefetchSummary
        y = torch.empty_like(x)
        recs = (PrefetchRecord * (steps * self.N))()
        sm = PrefetchSummary()
        call("moe_prefetch_run", self._h, steps, x.data_ptr(), y.data_ptr(),
             C.cast(recs, C.c_void_p), C.byref(sm), _stream(stream))
        names = ("cache_hit", "fetched_fresh", "evicted_and_fetched", "stream_through")
        records = [{"step": r.step, "layer": r.layer, "outcome": names[r.kind],
                    "victim": int(r.victim), "io_ms": r.io_ms, "h2d_start": r.h2d_start,
                    "h2d_end": r.h2d_end, "compute_start": r.compute_start,
                    "compute_end": r.compute_end} for r in recs]
        summary = {k: getattr(sm, k) for k, _ in PrefetchSummary._fields_}
        return y, records, summary

    @staticmethod
    def outcomes_jsonl(records) -> str:
        """prefetch_cache.cpp:206-217 outcomes_to_jsonl: one JSON object per access."""
        import json
        out = []
        for r in records:
            line = {"layer": r["layer"], "outcome": r["outcome"], "step": r["step"]}
            if r["outcome"] == "evicted_and_fetched":
                line["victim"] = r["victim"]
            out.append(json.dumps(line, sort_keys=True, separators=(",", ":")))
        return "".join(x + "\n" for x in out)

    def close(self):
        if getattr(self, "_h", None):
            call("moe_prefetch_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
