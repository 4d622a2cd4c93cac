"""2D prefetch with the Algorithm-1 CPU cache on real tiers:
a backing-store file (the SSD tier), pinned CPU blocks (cpu_size sections),
lookahead+1 HBM slots.  Prints one JSON line per cache size with the
reference's run_2d_schedule metrics (makespan, total stall, outcome counts,
bytes) measured on the CUDA-event timeline and the host I/O clock.

    python benchmarks/prefetch_bench.py [--layers 8 --steps 3 --tokens 16384]
"""
import argparse
import collections
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2205_10034_b200 import MoEConfig, MoELayer  # noqa: E402
from paper_2205_10034_b200.ring import Prefetch2D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--dff", type=int, default=8192)
    ap.add_argument("--lookahead", type=int, default=1)
    ap.add_argument("--cpu-sizes", type=int, nargs="+", default=[0, 4, 9])
    ap.add_argument("--dir", default=None, help="directory for the backing-store file")
    a = ap.parse_args()
    cfg = MoEConfig(a.experts, 2, a.d, a.dff, 1.25, a.tokens, torch.bfloat16)
    layer = MoELayer(cfg)
    x = layer.make_input(4)
    d = a.dir or tempfile.mkdtemp(prefix="moe_prefetch_", dir=os.getcwd())
    for cs in a.cpu_sizes:
        pf = Prefetch2D(layer, a.layers, a.lookahead, cs, os.path.join(d, f"store_{cs}.bin"),
                        threshold=1.0, beta=1.0, decay_steps=1, flush_period=a.steps, seed=5)
        pf.run(x, 1)  # warm-up (kernel attributes, first pinned allocations)
        torch.cuda.synchronize()
        _, recs, sm = pf.run(x, a.steps)
        counts = collections.Counter(r["outcome"] for r in recs)
        print(json.dumps({
            "bench": "prefetch_2d", "layers": a.layers, "steps": a.steps, "tokens": a.tokens,
            "experts": a.experts, "d_model": a.d, "d_ff": a.dff, "lookahead": a.lookahead,
            "cpu_size": cs, "section_bytes": sm["section_bytes"], "gpu_slots": sm["gpu_slots"],
            "makespan_ms": sm["makespan_ms"], "compute_total_ms": sm["compute_total_ms"],
            "stall_total_ms": sm["stall_total_ms"], "io_total_ms": sm["io_total_ms"],
            "bytes_read": sm["bytes_read"], "bytes_written": sm["bytes_written"],
            "h2d_bytes": sm["h2d_bytes"], "outcomes": dict(counts),
            "tokens_per_s": a.tokens * a.steps / (sm["makespan_ms"] / 1e3),
        }), flush=True)
        pf.close()


if __name__ == "__main__":
    main()
