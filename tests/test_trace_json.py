"""CPU: routing-trace export against the reference's own JSON
writer/reader (workload.cpp:68-119, golden vectors from oracle/_ref), and the
recorder's multi-rank gather over gloo (world_size 2)."""
import json
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

from mp_ranks import run_ranks

import oracle
from paper_2205_10034_b200 import moesim
from paper_2205_10034_b200._lib import ConfigError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


@pytest.mark.parametrize("ent", GOLD["trace_to_json"], ids=lambda e: str(e["args"]))
def test_trace_to_json_matches_reference_bytes(ent):
    seed, steps, ranks, experts, tokens, skew = ent["args"]
    if steps == 0:
        tr = moesim.RoutingTrace(0, ranks, experts, tokens, np.zeros((0, ranks, experts), np.uint64))
    else:  # counts from the CPU restatement (bit-exact with the reference, test_oracle_golden)
        c = oracle.gen_trace(seed, steps, ranks, experts, tokens, skew)
        tr = moesim.RoutingTrace(steps, ranks, experts, tokens, np.asarray(c, np.uint64))
    assert moesim.trace_to_json(tr) == ent["json"]
    back = moesim.trace_from_json(ent["json"])
    assert (back.steps, back.ranks, back.experts, back.tokens_per_rank) == (steps, ranks, experts, tokens)
    assert np.array_equal(back.counts.reshape(-1), np.asarray(tr.counts).reshape(-1))


@pytest.mark.parametrize("ent", GOLD["trace_from_json"], ids=lambda e: e["json"][:40])
def test_trace_from_json_errors_match_reference(ent):
    exp = ent["expected"]
    if "error" in exp:
        assert exp["error"] == 3  # ConfigError
        with pytest.raises(ConfigError) as ei:
            moesim.trace_from_json(ent["json"])
        assert str(ei.value) == exp["message"]
    else:
        tr = moesim.trace_from_json(ent["json"])
        assert tr.counts.reshape(-1).tolist() == exp["counts"]
        assert tr.tokens_per_rank == exp["tokens_per_rank"]




def _worker(rank, world, port, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        rec = moesim.RoutingTraceRecorder(experts=4, tokens=10, top_k=2, max_steps=3, device="cpu")
        for s in range(3):
            c1 = torch.tensor([s + rank, 10 - s - rank, 0, 0], dtype=torch.int32)
            c2 = torch.tensor([0, 0, 5, 5], dtype=torch.int32)
            rec.record({"count1": c1, "count2": c2})
        tr = rec.trace()
        q.put((rank, moesim.trace_to_json(tr)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_recorder_gathers_ranks_in_order():
    out = run_ranks(_worker, 2, timeout=120, is_ok=lambda m: m.startswith("{"))
    assert out[0] == out[1], out
    tr = moesim.trace_from_json(out[0])  # validates row sums = k*T
    assert (tr.steps, tr.ranks, tr.experts, tr.tokens_per_rank) == (3, 2, 4, 20)
    for s in range(3):
        for r in range(2):
            assert tr.counts[s, r].tolist() == [s + r, 10 - s - r, 5, 5]
