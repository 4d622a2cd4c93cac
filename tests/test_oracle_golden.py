"""CPU: pin the oracle (oracle/moe_oracle.c) against the reference's own outputs.

tests/golden/reference_golden.json was produced by running the reference
library compiled from /root/reference/proj (tests/golden/make_golden.py); the
cases are the ones its own tests pin (test_workload.cpp:72-133,
test_collectives.cpp:43-171, test_ring_offload.cpp:29-152) plus config-sized
ones.  When oracle/_ref is present (build container) the oracle is also
checked against the live reference on random cases.
"""
import ctypes as C

import numpy as np
import pytest

import oracle


def test_splitmix64_and_substreams(golden):
    for ent in golden["splitmix64"]:
        s = C.c_uint64(ent["seed"])
        got = [str(oracle.lib().oracle_splitmix64_next(C.byref(s))) for _ in ent["draws"]]
        assert got == ent["draws"]
    for ent in golden["substream_seed"]:
        assert str(oracle.substream_seed(*ent["args"])) == ent["value"]


def test_gen_trace_matches_reference(golden):
    for ent in golden["gen_trace"]:
        seed, steps, ranks, experts, tokens, skew = ent["args"]
        got = oracle.gen_trace(seed, steps, ranks, experts, tokens, skew)
        assert got.astype(np.int64).tolist() == ent["counts"], ent["args"]
        # conservation (test_workload.cpp:94-103)
        assert (got.sum(axis=2) == tokens).all()
        if "imbalance_ratio" in ent:
            assert oracle.imbalance_ratio(got) == ent["imbalance_ratio"]


def test_gen_trace_config_errors():
    with pytest.raises(ValueError):
        oracle.gen_trace(1, 1, 1, 0, 10, 0.0)  # experts = 0 (test_workload.cpp:105-107)
    with pytest.raises(ValueError):
        oracle.gen_trace(1, 1, 1, 4, 10, -1.0)


def test_imbalance_ratio(golden):
    for ent in golden["imbalance_ratio"]:
        assert oracle.imbalance_ratio(np.array(ent["counts"], dtype=np.uint64)) == ent["value"]
    with pytest.raises(ValueError):  # zero tokens -> ConfigError in the reference
        oracle.imbalance_ratio(np.zeros((1, 1, 2), dtype=np.uint64))


def _a2a(ranks, chunks):
    lens = np.array([len(c) for c in chunks], dtype=np.uint64)
    data = np.frombuffer(b"".join(chunks) or b"\0", dtype=np.uint8).copy()
    out_lens = np.zeros(len(chunks), dtype=np.uint64)
    out = np.zeros(max(1, int(lens.sum())), dtype=np.uint8)
    rc = oracle.lib().oracle_alltoall_flat(ranks, len(chunks), oracle.P(lens), oracle.P(data),
                                           oracle.P(out_lens), oracle.P(out))
    if rc:
        return {"error": rc}
    res, o = [], 0
    for ln in out_lens:
        res.append(out[o:o + int(ln)].tobytes().hex())
        o += int(ln)
    return {"chunks": res}


def test_alltoall_flat_matches_reference(golden):
    for ent in golden["alltoall_flat"]:
        got = _a2a(ent["ranks"], [bytes.fromhex(c) for c in ent["chunks"]])
        assert got == ent["expected"]


def test_alltoall_hierarchical_matches_reference(golden):
    """collectives.cpp:31-79 — delivery and per-phase hop stats, test_collectives.cpp:69-110."""
    for ent in golden["alltoall_hierarchical"]:
        chunks = [bytes.fromhex(c) for c in ent["chunks"]]
        lens = np.array([len(c) for c in chunks] or [0], dtype=np.uint64)
        data = np.frombuffer(b"".join(chunks) or b"\0", dtype=np.uint8).copy()
        out_lens = np.zeros(max(1, len(chunks)), dtype=np.uint64)
        out = np.zeros(max(1, int(lens.sum())), dtype=np.uint8)
        stats = np.zeros(14, dtype=np.uint64)
        rc = oracle.lib().oracle_alltoall_hierarchical(
            *ent["topo"], ent["ranks"], len(chunks), oracle.P(lens), oracle.P(data),
            oracle.P(out_lens), oracle.P(out), oracle.P(stats))
        if "error" in ent["expected"]:
            assert rc == ent["expected"]["error"], ent["topo"]
            continue
        assert rc == 0
        assert stats.tolist() == ent["expected"]["stats"], ent["topo"]
        assert _a2a(ent["ranks"], chunks)["chunks"] == ent["expected"]["chunks"]
        assert stats[6 + 5] == 0 and stats[3] == 0 and stats[5] == 0  # rails only


def test_fuse_split_match_reference(golden):
    for ent in golden["fuse_slices"]:
        slices = [bytes.fromhex(s) for s in ent["slices"]]
        n = len(slices)
        lens = np.array([len(s) for s in slices] or [0], dtype=np.uint64)
        data = np.frombuffer(b"".join(slices) or b"\0", dtype=np.uint8).copy()
        blob = np.zeros(max(1, int(lens.sum())), dtype=np.uint8)
        idx = np.zeros((max(n, 1), 3), dtype=np.uint64)
        rc = oracle.lib().oracle_fuse_slices(n, oracle.P(lens), oracle.P(data), oracle.P(blob),
                                             oracle.P(idx))
        if "error" in ent["expected"]:
            assert rc == ent["expected"]["error"]
            continue
        assert rc == 0
        assert blob[: int(lens[:n].sum())].tobytes().hex() == ent["expected"]["blob"]
        assert idx[:n].tolist() == ent["expected"]["index"]
    for ent in golden["split_blob"]:
        blob = bytes.fromhex(ent["blob"])
        index = ent["index"]
        b = np.frombuffer(blob or b"\0", dtype=np.uint8).copy()
        idx = np.array(index, dtype=np.uint64)
        out = np.zeros(max(1, len(blob)), dtype=np.uint8)
        rc = oracle.lib().oracle_split_blob(len(blob), oracle.P(b), len(index), oracle.P(idx),
                                            oracle.P(out))
        if "error" in ent["expected"]:
            assert rc == ent["expected"]["error"]
        else:
            assert rc == 0
            res, o = [], 0
            for (_, _, ln) in index:
                res.append(out[o:o + ln].tobytes().hex())
                o += ln
            assert res == ent["expected"]["slices"]


def test_ring_schedule_matches_reference(golden):
    for ent in golden["ring_schedule"]:
        n, k = ent["args"]
        ops = np.zeros((4 * max(n, 1) + 8, 4), dtype=np.int64)
        cnt, slots, cl = C.c_uint64(), C.c_uint32(), C.c_int()
        rc = oracle.lib().oracle_ring_schedule(n, k, oracle.P(ops), C.byref(cnt), C.byref(slots),
                                               C.byref(cl))
        if "error" in ent["expected"]:
            assert rc == ent["expected"]["error"]
            continue
        assert ops[: cnt.value].tolist() == ent["expected"]["ops"]
        assert slots.value == ent["expected"]["slots"]
        assert bool(cl.value) == ent["expected"]["clamped"]


def oracle_simulate(layers, slots, eb, db, comp, bw, lat):
    comp = np.array(comp, dtype=np.int64)
    ls, le, cs, ce = (np.zeros(layers, np.int64) for _ in range(4))
    mk, st, cp = C.c_int64(), C.c_int64(), C.c_int64()
    pk, bl = C.c_uint64(), C.c_uint64()
    rc = oracle.lib().oracle_ring_simulate(layers, slots, eb, db, oracle.P(comp), bw, lat,
                                           oracle.P(ls), oracle.P(le), oracle.P(cs),
                                           oracle.P(ce), C.byref(mk), C.byref(st), C.byref(cp),
                                           C.byref(pk), C.byref(bl))
    assert rc == 0
    return {"load_start": ls.tolist(), "load_end": le.tolist(), "compute_start": cs.tolist(),
            "compute_end": ce.tolist(), "makespan": mk.value, "stall": st.value,
            "copy_ns": cp.value, "peak_bytes": pk.value, "baseline_bytes": bl.value}


def test_ring_simulate_matches_reference(golden):
    for ent in golden["ring_simulate"]:
        a = ent["args"]
        assert oracle_simulate(*a) == ent["expected"], a


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built (no /root/reference)")
def test_oracle_vs_live_reference_random():
    rng = np.random.RandomState(1234)
    for _ in range(20):
        args = (int(rng.randint(0, 2**62)), int(rng.randint(1, 3)), int(rng.randint(1, 5)),
                int(rng.randint(1, 40)), int(rng.randint(0, 3000)), float(rng.choice([0, 0.5, 1.2, 2.0])))
        assert (oracle.gen_trace(*args) == oracle.gen_trace(*args, which="ref")).all()
