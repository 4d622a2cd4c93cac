"""CPU: the layer-step / ring timelines exported as the reference's trace-event
JSON (trace_export.cpp:28-58) -- semantically identical to what the compiled
reference's timeline_to_trace_json produces for the same Timeline, and valid
under its validate_trace_json; plus bench.py's restatement of the reference
ring model against the oracle's pinned ring_simulate."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle
from paper_2205_10034_b200 import moesim


def _tasks():
    ph = [("fwd.gate_gemm", 0.046), ("fwd.route", 0.024), ("fwd.dispatch", 0.048),
          ("fwd.ffn1", 0.507), ("bwd.combine_bwd", 0.074), ("bwd.wgrad_w1", 0.4941)]
    t = moesim.layer_step_timeline(ph, stream="rank0.compute")
    tl = {"load_start": [0.0, 38.6], "load_end": [38.6, 77.3], "compute_start": [38.6, 77.3],
          "compute_end": [45.8, 84.5]}
    r = moesim.ring_timeline(tl)
    return t + [moesim.TaskRecord(len(t) + x.id, x.label, x.stream, x.start, x.end) for x in r]


def test_layer_timeline_is_back_to_back():
    t = moesim.layer_step_timeline([("a", 1.0), ("b", 0.5)])
    assert [(x.start, x.end) for x in t] == [(0, 1000000), (1000000, 1500000)]


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built")
def test_trace_json_matches_compiled_reference():
    tasks = _tasks()
    ours = moesim.timeline_to_trace_json(tasks)
    r = oracle.ref()
    r.ref_timeline_trace_json.argtypes = [C.c_uint64, C.c_char_p, C.c_char_p, C.c_void_p,
                                          C.c_void_p, C.c_char_p, C.c_uint64,
                                          C.POINTER(C.c_uint64)]
    labels = b"".join(t.label.encode() + b"\0" for t in tasks)
    streams = b"".join(t.stream.encode() + b"\0" for t in tasks)
    st = np.array([t.start for t in tasks], np.int64)
    en = np.array([t.end for t in tasks], np.int64)
    buf = C.create_string_buffer(1 << 20)
    n = C.c_uint64(0)
    assert r.ref_timeline_trace_json(len(tasks), labels, streams, oracle.P(st), oracle.P(en),
                                     buf, 1 << 20, C.byref(n)) == 0
    assert json.loads(buf.value.decode()) == ours
    err = C.create_string_buffer(256)
    r.ref_validate_trace_json.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64]
    assert r.ref_validate_trace_json(json.dumps(ours).encode(), err, 256) == 0
    assert err.value == b""


def test_export_trace_roundtrip(tmp_path):
    p = tmp_path / "t.json"
    moesim.export_trace(_tasks(), str(p))
    assert json.loads(p.read_text()) == moesim.timeline_to_trace_json(_tasks())
    with pytest.raises(moesim.ConfigError):
        moesim.export_trace(_tasks(), str(tmp_path / "missing" / "t.json"))


@pytest.mark.parametrize("layers,slots,comp", [(12, 2, 7191497), (4, 2, 66136730), (5, 8, 1000),
                                               (24, 3, 5000000)])
def test_bench_ring_prediction_matches_oracle(layers, slots, comp):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    sec = 2148139008
    got = bench.ring_predicted(layers, slots, sec, [comp] * layers, 25e9, 2000)
    K = min(slots, layers)
    arr = {n: np.zeros(layers, np.int64) for n in ("ls", "le", "cs", "ce")}
    out = [C.c_int64(), C.c_int64(), C.c_int64(), C.c_uint64(), C.c_uint64()]
    cn = np.full(layers, comp, np.int64)
    rc = oracle.lib().oracle_ring_simulate(layers, slots, sec, 0, oracle.P(cn), 25 * 10**9, 2000,
                                           oracle.P(arr["ls"]), oracle.P(arr["le"]),
                                           oracle.P(arr["cs"]), oracle.P(arr["ce"]),
                                           *[C.byref(o) for o in out])
    assert rc == 0 and K >= 1
    assert got["makespan_ms"] == pytest.approx(out[0].value / 1e6, abs=1e-9)
    assert got["stall_ms"] == pytest.approx(out[1].value / 1e6, abs=1e-9)


def test_bench_c3_gate_bias_reproduces_gen_trace_skew():
    """bench.py c3: the calibrated gate bias makes top-1 choices of N(0, 1/9)
    logits follow the Zipf(1.2) distribution of gen_trace (workload.cpp:19-53)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    E = 32
    b = np.array(bench.zipf_gate_bias(E, 1.2), np.float32)
    z = np.random.default_rng(99).standard_normal((300000, E)).astype(np.float32) / 3 + b
    q = np.bincount(z.argmax(1), minlength=E) / len(z)
    ref = oracle.gen_trace(7, 1, 1, E, 300000, 1.2)[0, 0] / 300000.0
    assert np.abs(q - ref).max() < 0.01
    assert abs(q.max() * E / oracle.imbalance_ratio(oracle.gen_trace(7, 1, 1, E, 300000, 1.2)) - 1) < 0.02
