"""CPU: the Algorithm-1 CPU cache policy (moe_sparse_cache_*)
against the compiled reference's SparseCache (prefetch_cache.cpp:28-64):
outcome per access, victims, final hit-count snapshot, occupancy and decay
phase for the reference's own test cases (test_prefetch_cache.cpp:77-193) and
its randomized interpreter sweep (seed 4242), plus the config errors."""
import json
import os

import pytest

from paper_2205_10034_b200._lib import ConfigError
from paper_2205_10034_b200.moesim import SparseCache

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


@pytest.mark.parametrize("i", range(len(GOLD["sparse_cache"])))
def test_sparse_cache_matches_reference(i):
    ent = GOLD["sparse_cache"][i]
    cpu, thr, beta, k = ent["params"]
    exp = ent["expected"]
    if "error" in exp:
        assert exp["error"] == 3
        with pytest.raises(ConfigError, match=r"^cache\.(beta|decay_steps|threshold): "):
            SparseCache(cpu, thr, beta, k)
        return
    c = SparseCache(cpu, thr, beta, k)
    for op, kind, victim in zip(ent["ops"], exp["kinds"], exp["victims"]):
        if op < 0:
            c.end_step()
            continue
        got = c.access(op)
        assert got[0] == kind, (op, got, kind)
        if kind == 2:
            assert got[1] == victim
    occ, steps, snap = c.state()
    assert occ == exp["acc_caches"] and steps == exp["steps"]
    assert sorted(snap.items()) == [(int(b), h) for b, h in exp["snapshot"]]
    assert occ <= max(cpu, 0)


def test_reference_examples():
    """test_prefetch_cache.cpp:95-108: evict the coldest warm-enough block."""
    c = SparseCache(3, 1.0, 1.0, 1)
    for b in (1, 1, 1, 2):
        c.access(b)
    assert c.access(3) == (2, 2)
    _, _, snap = c.state()
    assert 2 not in snap and snap[3] == 1.0 and snap[1] == 3.0
