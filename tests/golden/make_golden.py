"""Generate tests/golden/*.json from the REFERENCE ITSELF.

Runs oracle/_ref/libmoesim_ref.so — the reference's own collectives.cpp,
workload.cpp, ring_offload.cpp, sim_engine.cpp and topology.cpp compiled from
/root/reference/proj by oracle/Makefile — on the cases its own tests pin
(test_workload.cpp, test_collectives.cpp, test_ring_offload.cpp,
acceptance_main.cpp) plus config-sized cases, and stores inputs + outputs.
The GPU box has no /root/reference; the fixtures travel instead.

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sm64(seed):
    s = C.c_uint64(seed)
    while True:
        yield int(oracle.ref().ref_splitmix64_next(C.byref(s)))


def random_payload(ranks, seed, max_len=16):
    """test_collectives.cpp:17-28 random_payload (chunk sizes and bytes from SplitMix64)."""
    g = sm64(seed)
    chunks = []
    for _ in range(ranks * ranks):
        n = next(g) % (max_len + 1)
        chunks.append(bytes(next(g) & 0xFF for _ in range(n)))
    return chunks


def ref_a2a(ranks, chunks):
    r = oracle.ref()
    lens = np.array([len(c) for c in chunks], dtype=np.uint64)
    data = np.frombuffer(b"".join(chunks) or b"\0", dtype=np.uint8).copy()
    out_lens = np.zeros(len(chunks), dtype=np.uint64)
    out = np.zeros(max(1, int(lens.sum())), dtype=np.uint8)
    rc = r.ref_alltoall_flat(ranks, len(chunks), oracle.P(lens), oracle.P(data),
                             oracle.P(out_lens), oracle.P(out))
    if rc:
        return {"error": rc}
    res, o = [], 0
    for ln in out_lens:
        res.append(out[o:o + int(ln)].tobytes().hex())
        o += int(ln)
    return {"chunks": res}


def ref_a2a_hier(topo, ranks, chunks):
    r = oracle.ref()
    lens = np.array([len(c) for c in chunks] or [0], dtype=np.uint64)
    data = np.frombuffer(b"".join(chunks) or b"\0", dtype=np.uint8).copy()
    out_lens = np.zeros(max(1, len(chunks)), dtype=np.uint64)
    out = np.zeros(max(1, int(lens.sum())), dtype=np.uint8)
    stats = np.zeros(14, dtype=np.uint64)
    rc = r.ref_alltoall_hierarchical(*topo, ranks, len(chunks), oracle.P(lens), oracle.P(data),
                                     oracle.P(out_lens), oracle.P(out), oracle.P(stats))
    if rc:
        return {"error": rc}
    res, o = [], 0
    for ln in out_lens[:len(chunks)]:
        res.append(out[o:o + int(ln)].tobytes().hex())
        o += int(ln)
    return {"chunks": res, "stats": [int(v) for v in stats]}


def ref_fuse(slices):
    r = oracle.ref()
    n = len(slices)
    lens = np.array([len(s) for s in slices] or [0], dtype=np.uint64)
    data = np.frombuffer(b"".join(slices) or b"\0", dtype=np.uint8).copy()
    blob = np.zeros(max(1, int(lens.sum())), dtype=np.uint8)
    idx = np.zeros((max(n, 1), 3), dtype=np.uint64)
    rc = r.ref_fuse_slices(n, oracle.P(lens), oracle.P(data), oracle.P(blob), oracle.P(idx))
    if rc:
        return {"error": rc}
    return {"blob": blob[: int(lens[:n].sum())].tobytes().hex(), "index": idx[:n].tolist()}


def ref_split(blob, index):
    r = oracle.ref()
    n = len(index)
    b = np.frombuffer(blob or b"\0", dtype=np.uint8).copy()
    idx = np.array(index or [[0, 0, 0]], dtype=np.uint64)
    out = np.zeros(max(1, len(blob)), dtype=np.uint8)
    rc = r.ref_split_blob(len(blob), oracle.P(b), n, oracle.P(idx), oracle.P(out))
    if rc:
        return {"error": rc}
    res, o = [], 0
    for (_, _, ln) in index:
        res.append(out[o:o + ln].tobytes().hex())
        o += ln
    return {"slices": res}


def ref_schedule(layers, slots):
    r = oracle.ref()
    ops = np.zeros((4 * layers + 8, 4), dtype=np.int64)
    n, k, cl = C.c_uint64(), C.c_uint32(), C.c_int()
    rc = r.ref_ring_schedule(layers, slots, oracle.P(ops), C.byref(n), C.byref(k), C.byref(cl))
    if rc:
        return {"error": rc}
    return {"ops": ops[: n.value].tolist(), "slots": k.value, "clamped": bool(cl.value)}


def ref_simulate(layers, slots, expert_bytes, dense_bytes, compute_ns, bw, lat):
    r = oracle.ref()
    comp = np.array(compute_ns, dtype=np.int64)
    ls, le, cs, ce = (np.zeros(layers, np.int64) for _ in range(4))
    mk, st, cp = C.c_int64(), C.c_int64(), C.c_int64()
    pk, bl = C.c_uint64(), C.c_uint64()
    rc = r.ref_ring_simulate(layers, slots, expert_bytes, dense_bytes, oracle.P(comp), bw, lat,
                             oracle.P(ls), oracle.P(le), oracle.P(cs), oracle.P(ce), C.byref(mk),
                             C.byref(st), C.byref(cp), C.byref(pk), C.byref(bl))
    if rc:
        return {"error": rc}
    return {"load_start": ls.tolist(), "load_end": le.tolist(), "compute_start": cs.tolist(),
            "compute_end": ce.tolist(), "makespan": mk.value, "stall": st.value,
            "copy_ns": cp.value, "peak_bytes": pk.value, "baseline_bytes": bl.value}


def ref_trace_to_json(steps, ranks, experts, tokens, counts):
    r = oracle.ref()
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64).reshape(-1))
    buf = C.create_string_buffer(1 << 22)
    n = C.c_uint64(0)
    rc = r.ref_trace_to_json(C.c_uint32(steps), C.c_uint32(ranks), C.c_uint32(experts),
                             C.c_uint64(tokens), oracle.P(c) if c.size else None, buf,
                             C.c_uint64(len(buf)), C.byref(n))
    assert rc == 0, rc
    return buf.value.decode()


def ref_trace_from_json(text):
    r = oracle.ref()
    st, rk, ex = C.c_uint32(0), C.c_uint32(0), C.c_uint32(0)
    tok = C.c_uint64(0)
    counts = np.zeros(1 << 16, dtype=np.uint64)
    err = C.create_string_buffer(512)
    rc = r.ref_trace_from_json(text.encode(), C.byref(st), C.byref(rk), C.byref(ex), C.byref(tok),
                               oracle.P(counts), C.c_uint64(counts.size), err, C.c_uint64(512))
    if rc:
        return {"error": rc, "message": err.value.decode()}
    n = st.value * rk.value * ex.value
    return {"steps": st.value, "ranks": rk.value, "experts": ex.value, "tokens_per_rank": tok.value,
            "counts": counts[:n].astype(np.int64).tolist()}


def ref_sparse_cache(params, ops):
    r = oracle.ref()
    n = len(ops)
    o = np.asarray(ops, dtype=np.int64)
    kinds = np.zeros(max(n, 1), dtype=np.int32)
    victims = np.zeros(max(n, 1), dtype=np.uint64)
    sb = np.zeros(4096, dtype=np.uint64)
    sh = np.zeros(4096, dtype=np.float64)
    sn, acc, st = C.c_uint64(0), C.c_uint64(0), C.c_uint32(0)
    rc = r.ref_sparse_cache_run(C.c_uint64(params[0]), C.c_double(params[1]), C.c_double(params[2]),
                                C.c_uint32(params[3]), oracle.P(o), C.c_uint64(n), oracle.P(kinds),
                                oracle.P(victims), oracle.P(sb), oracle.P(sh), C.c_uint64(4096),
                                C.byref(sn), C.byref(acc), C.byref(st))
    if rc:
        return {"error": rc}
    return {"kinds": kinds[:n].tolist(), "victims": victims[:n].astype(np.int64).tolist(),
            "snapshot": [[int(sb[i]), float(sh[i])] for i in range(sn.value)],
            "acc_caches": acc.value, "steps": st.value}


def main():
    assert oracle.ref() is not None, "build the reference first: make -C oracle ref"
    gold = {"source": "oracle/_ref/libmoesim_ref.so built from /root/reference/proj (see oracle/Makefile)"}

    # rng.hpp:19-42
    gold["splitmix64"] = [{"seed": s, "draws": [str(v) for v, _ in zip(sm64(s), range(8))]}
                          for s in (0, 1, 7, 0xC0113C7, 2**64 - 1)]
    gold["substream_seed"] = [{"args": [s, st, r], "value": str(int(oracle.ref().ref_substream_seed(s, st, r)))}
                              for s, st, r in ((7, 0, 0), (11, 2, 1), (13, 0, 15), (2**63 + 5, 7, 3))]

    # workload.cpp:19-66 — test_workload.cpp:72-84 cases + config-sized ones
    traces = []
    for args in ((7, 1, 2, 4, 100, 0.0), (11, 3, 2, 8, 64, 1.2), (7, 2, 3, 1, 50, 1.5),
                 (7, 2, 2, 4, 0, 0.0), (42, 4, 4, 16, 256, 0.9), (5, 3, 5, 7, 129, 2.0),
                 (13, 1, 16, 16, 4096, 0.5),          # scenarios/alltoall_bench.json
                 (3, 1, 8, 64, 65536, 0.0),           # c2-scale uniform
                 (3, 1, 8, 32, 65536, 1.2)):          # c3-scale skewed
        c = oracle.gen_trace(*args, which="ref")
        ent = {"args": list(args), "counts": c.astype(np.int64).tolist()}
        if c.sum():
            ent["imbalance_ratio"] = oracle.imbalance_ratio(c, "ref")
        traces.append(ent)
    gold["gen_trace"] = traces
    gold["imbalance_ratio"] = [
        {"counts": [[[90, 10]]], "value": 1.8}, {"counts": [[[50, 50]]], "value": 1.0},
        {"counts": [[[10]]], "value": 1.0}]
    for ent in gold["imbalance_ratio"]:
        ent["value"] = oracle.imbalance_ratio(np.array(ent["counts"], dtype=np.uint64), "ref")

    # collectives.cpp:10-21 — test_collectives.cpp:43-66 + acceptance crit 3 style
    a2a = [{"ranks": 2, "chunks": [b"a".hex(), b"b".hex(), b"c".hex(), b"d".hex()]},
           {"ranks": 1, "chunks": [bytes([1, 2, 3]).hex()]}]
    a2a.append({"ranks": 4, "chunks": [c.hex() for c in random_payload(4, 99)]})
    for r, seed in ((3, 5), (8, 1234), (5, 0xC0113C7)):
        a2a.append({"ranks": r, "chunks": [c.hex() for c in random_payload(r, seed, 64)]})
    a2a.append({"ranks": 2, "chunks": ["aa", "bb", "cc"]})  # non-square -> invalid_argument
    for ent in a2a:
        ent["expected"] = ref_a2a(ent["ranks"], [bytes.fromhex(c) for c in ent["chunks"]])
    gold["alltoall_flat"] = a2a

    # collectives.cpp:31-79 — test_collectives.cpp:69-110
    hier = [{"topo": [1, 1, 4], "ranks": 4, "chunks": [c.hex() for c in random_payload(4, 5)]},
            {"topo": [1, 2, 2], "ranks": 4,
             "chunks": [bytes([s_, d_]).hex() for s_ in range(4) for d_ in range(4)]}]
    seed = 1
    for cl in (1, 2):
        for nd in (1, 2):
            for gp in (1, 2, 3, 4):
                for _ in range(5):
                    R = cl * nd * gp
                    hier.append({"topo": [cl, nd, gp], "ranks": R,
                                 "chunks": [c.hex() for c in random_payload(R, seed)]})
                    seed += 1
    hier.append({"topo": [2, 2, 4], "ranks": 16,
                 "chunks": [c.hex() for c in random_payload(16, 77, 300)]})
    hier.append({"topo": [1, 2, 2], "ranks": 3, "chunks": [c.hex() for c in random_payload(3, 1)]})
    hier.append({"topo": [1, 2, 2], "ranks": 2, "chunks": ["aa", "bb", "cc"]})
    hier.append({"topo": [0, 2, 2], "ranks": 4, "chunks": [c.hex() for c in random_payload(4, 2)]})
    hier.append({"topo": [1, 1, 0], "ranks": 0, "chunks": []})
    for ent in hier:
        ent["expected"] = ref_a2a_hier(ent["topo"], ent["ranks"],
                                       [bytes.fromhex(c) for c in ent["chunks"]])
    gold["alltoall_hierarchical"] = hier

    # collectives.cpp:88-118 — test_collectives.cpp:136-171
    fuse = [[bytes([1, 2, 3])], [bytes([1, 2, 3]), b"", bytes([4, 5, 6, 7, 8])], []]
    g = sm64(17)
    for _ in range(6):
        sl = []
        for _ in range(1 + next(g) % 8):
            sl.append(bytes(next(g) & 0xFF for _ in range(next(g) % 12)))
        fuse.append(sl)
    gold["fuse_slices"] = [{"slices": [s.hex() for s in sl], "expected": ref_fuse(sl)} for sl in fuse]
    split = [
        {"blob": bytes([1, 2]).hex(), "index": [[0, 0, 2]]},
        {"blob": bytes([1, 2, 0]).hex(), "index": [[0, 0, 2]]},      # longer blob -> error
        {"blob": bytes([1, 2]).hex(), "index": [[0, 1, 2]]},         # gap -> error
        {"blob": bytes(range(8)).hex(), "index": [[0, 0, 3], [1, 3, 0], [2, 3, 5]]},
    ]
    for ent in split:
        ent["expected"] = ref_split(bytes.fromhex(ent["blob"]), ent["index"])
    gold["split_blob"] = split

    # ring_offload.cpp:31-117 — test_ring_offload.cpp:29-152, scenarios/infer_ring.json
    gold["ring_schedule"] = [{"args": [n, k], "expected": ref_schedule(n, k)}
                             for n, k in ((1, 1), (3, 1), (4, 2), (3, 10), (24, 2), (12, 2), (4, 0))]
    sec = 1_000_000_000
    sims = [
        (24, 2, 1000, 0, [2 * sec] * 24, 1000, 0),
        (5, 2, 0, 0, [3 * sec] * 5, 1000, 0),
        (6, 6, 1000, 0, [2 * sec] * 6, 1000, 0),
        (5, 1, 800, 0, [sec] * 5, 1000, 0),
        (5, 3, 800, 0, [sec] * 5, 1000, 0),
        (8, 3, 5000, 0, [sec] * 8, 1000, 0),
        (24, 2, 50_000_000, 120_000_000, [2_500_000] * 24, 25_000_000_000, 2000),
        (12, 2, 2_147_483_648, 1_000_000, [40_000_000 + 1_000_000 * i for i in range(12)],
         55_000_000_000, 2000),
    ]
    gold["ring_simulate"] = [{"args": list(a[:4]) + [a[4], a[5], a[6]],
                              "expected": ref_simulate(*a)} for a in sims]

    # workload.cpp:68-119 — routing-trace JSON (schemas/routing_trace.schema.json)
    tj = []
    for args in ((7, 1, 2, 4, 100, 0.0), (11, 3, 2, 8, 64, 1.2), (5, 2, 3, 5, 33, 0.7)):
        c = oracle.gen_trace(*args, which="ref")
        tj.append({"args": list(args), "json": ref_trace_to_json(args[1], args[2], args[3], args[4], c)})
    tj.append({"args": [0, 0, 1, 1, 0, 0.0], "json": ref_trace_to_json(0, 1, 1, 0, [])})
    gold["trace_to_json"] = tj
    bad = [
        '{"steps":1,"ranks":1,"experts":2,"counts":[[[1,1]]]}',                         # missing tokens
        '{"steps":2,"ranks":1,"experts":2,"tokens_per_rank":2,"counts":[[[1,1]]]}',     # steps
        '{"steps":1,"ranks":2,"experts":2,"tokens_per_rank":2,"counts":[[[1,1]]]}',     # ranks
        '{"steps":1,"ranks":1,"experts":3,"tokens_per_rank":2,"counts":[[[1,1]]]}',     # experts
        '{"steps":1,"ranks":1,"experts":2,"tokens_per_rank":3,"counts":[[[1,1]]]}',     # row sum
        '{"steps":1,"ranks":1,"experts":2,"tokens_per_rank":2,"counts":[[[2,0]]],"schema_version":1}',
    ]
    gold["trace_from_json"] = [{"json": t, "expected": ref_trace_from_json(t)} for t in bad]

    # prefetch_cache.cpp:28-64 — test_prefetch_cache.cpp:77-193 cases + random sweeps
    sc = [
        {"params": [4, 1.0, 1.0, 1], "ops": [100]},
        {"params": [4, 1.0, 1.0, 1], "ops": [100, 100]},
        {"params": [3, 1.0, 1.0, 1], "ops": [1, 1, 1, 2, 3]},
        {"params": [3, 5.0, 1.0, 1], "ops": [1, 1, 1, 2, 3]},
        {"params": [0, 1.0, 1.0, 1], "ops": [i % 3 for i in range(10)]},
        {"params": [1, 1.0, 1.0, 1], "ops": [i % 3 for i in range(10)]},
        {"params": [4, 1.0, 0.5, 2], "ops": [7, 7, 7, 7, -1, -1]},
        {"params": [4, 1.0, 0.25, 3], "ops": [7, -1]},
        {"params": [2, 0.0, 1.0, 1], "ops": [5, 3, 3, 9, 5]},          # tie-breaking / threshold 0
    ]
    g = sm64(4242)
    for _ in range(40):
        cpu = next(g) % 9
        thr = float(next(g) % 6)
        beta = 1.0 if next(g) % 2 == 0 else 0.5 + 0.0625 * (next(g) % 8)
        k = (1, 2, 5)[next(g) % 3]
        uni = 1 + next(g) % 12
        ops = []
        for _ in range(200):
            ops.append(-1 if next(g) % 8 == 0 else int(next(g) % uni))
        sc.append({"params": [cpu, thr, beta, k], "ops": ops})
    sc.append({"params": [4, 1.0, 0.0, 1], "ops": [1]})   # beta 0 -> ConfigError
    sc.append({"params": [4, 1.0, 1.0, 0], "ops": [1]})   # decay_steps 0 -> ConfigError
    sc.append({"params": [4, -1.0, 1.0, 1], "ops": [1]})  # threshold < 0 -> ConfigError
    for ent in sc:
        ent["expected"] = ref_sparse_cache(ent["params"], ent["ops"])
    gold["sparse_cache"] = sc

    with open(os.path.join(OUT, "reference_golden.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(OUT, "reference_golden.json"))


if __name__ == "__main__":
    main()
