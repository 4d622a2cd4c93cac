"""Python mirror of the reference's moesim:: functions on the path.

Same names, argument meaning and error behaviour as
/root/reference/proj/core/include/moesim/{collectives,workload,ring_offload}.hpp,
executed by libmoe_b200.so on the GPU (host buffers in, host buffers out — the
reference's value-semantics calling convention).  Chunks are ``bytes``.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import ConfigError, SliceIndexEntry, call, lib  # noqa: F401

Chunk = bytes


@dataclass
class ShardedPayload:
    """collectives.hpp:19-33 — square R x R chunk matrix, row-major [src][dst]."""
    ranks: int = 0
    chunks: List[bytes] = field(default_factory=list)

    @staticmethod
    def make(ranks: int) -> "ShardedPayload":
        return ShardedPayload(ranks, [b""] * (ranks * ranks))

    def at(self, src: int, dst: int) -> bytes:
        return self.chunks[src * self.ranks + dst]

    def set(self, src: int, dst: int, chunk: bytes) -> None:
        self.chunks[src * self.ranks + dst] = bytes(chunk)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else None


def alltoall_flat(payload: ShardedPayload) -> ShardedPayload:
    """collectives.cpp:10-21: chunks'[i][j] = chunks[j][i]; non-square -> ValueError."""
    n = len(payload.chunks)
    lens = _u64([len(c) for c in payload.chunks])
    data = np.frombuffer(b"".join(payload.chunks), dtype=np.uint8).copy()
    out_lens = np.zeros(n, dtype=np.uint64)
    out = np.zeros(max(int(lens.sum()), 1), dtype=np.uint8)
    call("moesim_alltoall_flat", payload.ranks, n, _ptr(lens), _ptr(data), _ptr(out_lens),
         _ptr(out))
    res = ShardedPayload.make(payload.ranks)
    o = 0
    for i in range(n):
        ln = int(out_lens[i])
        res.chunks[i] = out[o:o + ln].tobytes()
        o += ln
    return res


LINK_CLASSES = ("nvlink", "pcie", "ssd_io", "tor", "leaf", "spin")  # topology.hpp:15


@dataclass
class Topology:
    """topology.hpp:37-60 shape (clusters x nodes_per_cluster x gpus_per_node);
    zero dimensions raise ConfigError like the reference constructor."""
    clusters: int
    nodes_per_cluster: int
    gpus_per_node: int

    def __post_init__(self):
        for name in ("clusters", "nodes_per_cluster", "gpus_per_node"):
            if getattr(self, name) < 1:
                raise ConfigError(f"topology.{name}: must be >= 1")

    def total_gpus(self) -> int:
        return self.clusters * self.nodes_per_cluster * self.gpus_per_node


@dataclass
class AlltoAllStats:
    """collectives.hpp:38-47; hop lists are indexed like LINK_CLASSES."""
    phase1_hops: List[int] = field(default_factory=lambda: [0] * 6)
    phase2_hops: List[int] = field(default_factory=lambda: [0] * 6)
    phase1_transfers: int = 0
    phase2_transfers: int = 0

    def hops(self, link: str) -> int:
        i = LINK_CLASSES.index(link)
        return self.phase1_hops[i] + self.phase2_hops[i]


def alltoall_hierarchical(payload: ShardedPayload, topology: Topology,
                          stats: Optional[AlltoAllStats] = None) -> ShardedPayload:
    """collectives.cpp:31-79: rail-aware two-phase all-to-all (both phases on the
    GPU); delivers alltoall_flat's result and accumulates hop counts in stats."""
    n = len(payload.chunks)
    lens = _u64([len(c) for c in payload.chunks])
    data = np.frombuffer(b"".join(payload.chunks), dtype=np.uint8).copy()
    out_lens = np.zeros(n, dtype=np.uint64)
    out = np.zeros(max(int(lens.sum()), 1), dtype=np.uint8)
    st = np.zeros(14, dtype=np.uint64)
    call("moesim_alltoall_hierarchical", topology.clusters, topology.nodes_per_cluster,
         topology.gpus_per_node, payload.ranks, n, _ptr(lens), _ptr(data), _ptr(out_lens),
         _ptr(out), _ptr(st))
    if stats is not None:
        for i in range(6):
            stats.phase1_hops[i] += int(st[i])
            stats.phase2_hops[i] += int(st[6 + i])
        stats.phase1_transfers += int(st[12])
        stats.phase2_transfers += int(st[13])
    res = ShardedPayload.make(payload.ranks)
    o = 0
    for i in range(n):
        ln = int(out_lens[i])
        res.chunks[i] = out[o:o + ln].tobytes()
        o += ln
    return res


@dataclass
class FusedBlob:
    blob: bytes
    index: List[tuple]  # (slice_id, offset, length)


def fuse_slices(slices: Sequence[bytes]) -> FusedBlob:
    """collectives.cpp:88-98; empty list -> ValueError."""
    n = len(slices)
    lens = _u64([len(s) for s in slices])
    data = np.frombuffer(b"".join(slices), dtype=np.uint8).copy()
    blob = np.zeros(max(int(lens.sum()) if n else 0, 1), dtype=np.uint8)
    idx = (SliceIndexEntry * max(n, 1))()
    call("moesim_fuse_slices", n, _ptr(lens) if n else None, _ptr(data), _ptr(blob),
         C.cast(idx, C.c_void_p))
    total = int(lens.sum()) if n else 0
    return FusedBlob(blob[:total].tobytes(),
                     [(idx[i].slice_id, idx[i].offset, idx[i].length) for i in range(n)])


def split_blob(blob: bytes, index: Sequence[tuple]) -> List[bytes]:
    """collectives.cpp:100-118; non-contiguous / non-covering index -> ValueError."""
    n = len(index)
    idx = (SliceIndexEntry * max(n, 1))()
    for i, (sid, off, ln) in enumerate(index):
        idx[i].slice_id, idx[i].offset, idx[i].length = sid, off, ln
    b = np.frombuffer(bytes(blob), dtype=np.uint8).copy()
    out = np.zeros(max(len(blob), 1), dtype=np.uint8)
    call("moesim_split_blob", len(blob), _ptr(b), n, C.cast(idx, C.c_void_p), _ptr(out))
    res, o = [], 0
    for (_, _, ln) in index:
        res.append(out[o:o + ln].tobytes())
        o += ln
    return res


@dataclass
class RoutingTrace:
    """workload.hpp:14-30: counts[step][rank][expert] (uint64)."""
    steps: int
    ranks: int
    experts: int
    tokens_per_rank: int
    counts: np.ndarray

    def at(self, s: int, r: int, e: int) -> int:
        return int(self.counts[s, r, e])

    def expert_total(self, e: int) -> int:
        return int(self.counts[:, :, e].sum())


def gen_trace(seed: int, steps: int, ranks: int, experts: int, tokens_per_rank: int,
              skew: float) -> RoutingTrace:
    """workload.cpp:19-53 (device-generated, bit-identical)."""
    counts = np.zeros((steps, ranks, max(experts, 1)), dtype=np.uint64)
    call("moesim_gen_trace", seed, steps, ranks, experts, tokens_per_rank, float(skew),
         counts.ctypes.data_as(C.c_void_p))
    return RoutingTrace(steps, ranks, experts, tokens_per_rank, counts[:, :, :experts])


def imbalance_ratio(trace: RoutingTrace) -> float:
    """workload.cpp:55-66; zero tokens -> ConfigError."""
    counts = np.ascontiguousarray(trace.counts, dtype=np.uint64)
    out = C.c_double(0.0)
    call("moesim_imbalance_ratio", trace.steps, trace.ranks, trace.experts,
         counts.ctypes.data_as(C.c_void_p) if counts.size else None, C.byref(out))
    return out.value


def trace_to_json(trace: RoutingTrace) -> str:
    """workload.cpp:68-85 (schemas/routing_trace.schema.json): the same document
    the reference's trace_to_json(...).dump() writes — compact, keys sorted."""
    counts = np.asarray(trace.counts, dtype=np.uint64).reshape(trace.steps, trace.ranks, trace.experts)
    doc = {"schema_version": 1, "steps": int(trace.steps), "ranks": int(trace.ranks),
           "experts": int(trace.experts), "tokens_per_rank": int(trace.tokens_per_rank),
           "counts": counts.astype(np.int64).tolist()}
    return json.dumps(doc, sort_keys=True, separators=(",", ":"))


def trace_from_json(doc) -> RoutingTrace:
    """workload.cpp:87-119: validate and load a routing trace (str or dict);
    malformed documents raise ConfigError with the reference's messages."""
    if isinstance(doc, (str, bytes)):
        doc = json.loads(doc)
    for key in ("steps", "ranks", "experts", "tokens_per_rank", "counts"):
        if key not in doc:
            raise ConfigError(f"trace.{key}: missing field")
    steps, ranks, experts = int(doc["steps"]), int(doc["ranks"]), int(doc["experts"])
    tokens = int(doc["tokens_per_rank"])
    counts = doc["counts"]
    out = np.zeros((steps, ranks, experts), dtype=np.uint64)
    if not isinstance(counts, list) or len(counts) != steps:
        raise ConfigError("trace.counts: expected one entry per step")
    for si in range(steps):
        by_rank = counts[si]
        if not isinstance(by_rank, list) or len(by_rank) != ranks:
            raise ConfigError("trace.counts: expected one row per rank")
        for ri in range(ranks):
            row = by_rank[ri]
            if not isinstance(row, list) or len(row) != experts:
                raise ConfigError("trace.counts: expected one count per expert")
            out[si, ri, :] = row
            if sum(int(v) for v in row) != tokens:
                raise ConfigError("trace.counts: row sum does not match tokens_per_rank")
    return RoutingTrace(steps, ranks, experts, tokens, out)


class RoutingTraceRecorder:
    """Measured routing -> RoutingTrace: per step, the device
    routing's pre-drop assignment counts (count1 + count2 of moe_route /
    moe_layer_forward) are appended on the device, so recording adds no host
    synchronisation; `trace()` gathers all EP ranks (rank order) and returns the
    reference's [step][rank][expert] trace that `WorkloadConfig::trace_file`
    (scenario.cpp:67-80) can replay. tokens_per_rank = k * T (every token is
    routed k times)."""

    def __init__(self, experts: int, tokens: int, top_k: int, max_steps: int, device=None):
        import torch
        self.E, self.T, self.k = experts, tokens, top_k
        self.buf = torch.zeros(max_steps, experts, dtype=torch.int64, device=device or "cuda")
        self.steps = 0

    def record(self, routing) -> None:
        """routing: the dict returned by MoELayer.forward(..., routing=True) or route()."""
        if self.steps >= self.buf.shape[0]:
            raise ConfigError("trace.steps: recorder is full")
        c = routing["count1"].to(self.buf.dtype)
        if self.k == 2:
            c = c + routing["count2"].to(self.buf.dtype)
        self.buf[self.steps].copy_(c, non_blocking=True)
        self.steps += 1

    def trace(self, group=None) -> RoutingTrace:
        import torch
        import torch.distributed as dist
        mine = self.buf[: self.steps]
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            parts = [torch.empty_like(mine) for _ in range(dist.get_world_size(group))]
            dist.all_gather(parts, mine, group=group)
            allr = torch.stack(parts, dim=1)  # [step][rank][expert]
        else:
            allr = mine.unsqueeze(1)
        counts = allr.cpu().numpy().astype(np.uint64)
        return RoutingTrace(self.steps, counts.shape[1], self.E, self.k * self.T, counts)


class GradBuckets:
    """Gradient-bucket fusion (moe_grad_buckets_*) with the
    semantics of make_gradient_buckets + GradBucket (collectives.cpp:120-162):
    ids in layer order are registered in reverse into buckets of <= capacity;
    push(id) returns the bucket index it flushed (ids in registration order via
    ids(b)) or None while held.  With `grads` (fp32 device tensors, same order
    as ids) a flush packs, all-reduces over `ep` (NCCL) and unpacks x `scale`
    on the stream; without, it is bookkeeping only (CPU-usable)."""

    def __init__(self, ids_layer_order: Sequence[int], capacity: int, grads=None, ep=None,
                 scale: float = 1.0):
        n = len(ids_layer_order)
        self._ids = (C.c_uint64 * max(n, 1))(*ids_layer_order)
        gp = nm = None
        self._grads = list(grads) if grads is not None else None
        if grads is not None:
            assert len(grads) == n
            for g in grads:
                assert g.dtype.is_floating_point and g.element_size() == 4 and g.is_contiguous()
            gp = (C.c_void_p * max(n, 1))(*[g.data_ptr() for g in grads])
            nm = (C.c_uint64 * max(n, 1))(*[g.numel() for g in grads])
        h = C.c_void_p()
        call("moe_grad_buckets_create", ep.comm if ep is not None else None, n,
             C.cast(self._ids, C.c_void_p), C.cast(gp, C.c_void_p) if gp else None,
             C.cast(nm, C.c_void_p) if nm else None, capacity, float(scale), C.byref(h))
        self._h = h

    def __len__(self) -> int:
        return int(lib.moe_grad_buckets_count(self._h))

    def ids(self, b: int) -> List[int]:
        out = (C.c_uint64 * 4096)()
        n = C.c_uint32(0)
        call("moe_grad_buckets_ids", self._h, b, C.cast(out, C.c_void_p), 4096, C.byref(n))
        return [int(out[i]) for i in range(n.value)]

    def push(self, grad_id: int, stream=None) -> Optional[int]:
        from .layer import _stream
        f = C.c_int32(-1)
        call("moe_grad_buckets_push", self._h, grad_id,
             _stream(stream) if self._grads is not None else None, C.byref(f))
        return None if f.value < 0 else int(f.value)

    def reset(self) -> None:
        call("moe_grad_buckets_reset", self._h)

    def close(self) -> None:
        if getattr(self, "_h", None):
            call("moe_grad_buckets_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


CACHE_HIT, FETCHED_FRESH, EVICTED_AND_FETCHED, STREAM_THROUGH = 0, 1, 2, 3
CACHE_KIND_NAMES = ("cache_hit", "fetched_fresh", "evicted_and_fetched", "stream_through")


class SparseCache:
    """prefetch_cache.hpp:43-83 SparseCache over moe_sparse_cache_* (Algorithm-1
    CPU cache policy). access(block) -> (kind, victim); kind names as
    access_kind_name (prefetch_cache.cpp:16-24)."""

    def __init__(self, cpu_size: int, threshold: float = 1.0, beta: float = 1.0,
                 decay_steps: int = 1):
        from ._lib import CacheParams
        p = CacheParams(cpu_size, float(threshold), float(beta), decay_steps)
        h = C.c_void_p()
        call("moe_sparse_cache_create", C.byref(p), C.byref(h))
        self._h = h

    def access(self, block: int):
        from ._lib import CacheAccess
        out = CacheAccess()
        call("moe_sparse_cache_access", self._h, block, C.byref(out))
        return int(out.kind), int(out.victim)

    def end_step(self) -> None:
        call("moe_sparse_cache_end_step", self._h)

    def state(self):
        """(occupancy, steps, {block: hit count}) — hits_snapshot() is the dict."""
        occ, st, n = C.c_uint64(0), C.c_uint32(0), C.c_uint64(0)
        call("moe_sparse_cache_state", self._h, C.byref(occ), C.byref(st), None, None, 0, C.byref(n))
        blocks = (C.c_uint64 * max(n.value, 1))()
        hits = (C.c_double * max(n.value, 1))()
        call("moe_sparse_cache_state", self._h, None, None, C.cast(blocks, C.c_void_p),
             C.cast(hits, C.c_void_p), n.value, C.byref(n))
        return occ.value, st.value, {int(blocks[i]): float(hits[i]) for i in range(n.value)}

    def hit_count(self, block: int) -> float:
        return self.state()[2].get(block, 0.0)

    def close(self) -> None:
        if getattr(self, "_h", None):
            call("moe_sparse_cache_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


LOAD, COMPUTE, RELEASE = 0, 1, 2


@dataclass
class RingOp:
    kind: int
    layer: int
    slot: int
    waits_release_of: Optional[int]


@dataclass
class RingSchedule:
    ops: List[RingOp]
    slots: int
    clamped: bool


def build_schedule(num_layers: int, ring_slots: int) -> RingSchedule:
    """ring_offload.cpp:31-50; ring_slots == 0 or num_layers == 0 -> ConfigError."""
    cap = 3 * max(num_layers, 1) + max(num_layers, 1)
    ops = np.zeros((cap, 4), dtype=np.int64)
    n = C.c_uint64(0)
    slots = C.c_uint32(0)
    clamped = C.c_int(0)
    call("moesim_ring_build_schedule", num_layers, ring_slots, ops.ctypes.data_as(C.c_void_p),
         cap, C.byref(n), C.byref(slots), C.byref(clamped))
    res = [RingOp(int(k), int(l), int(s), None if w < 0 else int(w))
           for k, l, s, w in ops[: n.value]]
    return RingSchedule(res, slots.value, bool(clamped.value))


# ------------------------------------------------------------ timelines ----
@dataclass
class TaskRecord:
    """sim_engine.hpp:28-34 TaskRecord (times in ns)."""
    id: int
    label: str
    stream: str
    start: int
    end: int


def timeline_to_trace_json(tasks: Sequence[TaskRecord]) -> dict:
    """trace_export.cpp:28-50 timeline_to_trace_json: one thread_name metadata
    event per stream (streams in name order, tid = that order), then one
    complete ("X") event per task in submission order, times in us."""
    tids = {name: i for i, name in enumerate(sorted({t.stream for t in tasks}))}
    events = [{"args": {"name": n}, "name": "thread_name", "ph": "M", "pid": 1, "tid": i}
              for n, i in tids.items()]
    for t in tasks:
        events.append({"args": {"task_id": t.id}, "dur": (t.end - t.start) / 1000.0,
                       "name": t.label, "ph": "X", "pid": 1, "tid": tids[t.stream],
                       "ts": t.start / 1000.0})
    return {"displayTimeUnit": "ns", "traceEvents": events}


def export_trace(tasks: Sequence[TaskRecord], path: str) -> None:
    """trace_export.cpp:52-57 export_trace (ConfigError on an unwritable path)."""
    import json
    try:
        with open(path, "w") as f:
            f.write(json.dumps(timeline_to_trace_json(tasks), indent=2, sort_keys=True) + "\n")
    except OSError as e:
        raise ConfigError(f"trace: cannot open '{path}' for writing") from e


def layer_step_timeline(phases: Sequence[tuple], stream: str = "compute",
                        t0_ns: int = 0) -> List[TaskRecord]:
    """Timeline of one layer step from its per-phase CUDA-event durations
    (MoELayer.phase_times(), in launch order; the phases of one call are back
    to back on the launch stream, so start = running sum).  phases: (label, ms)."""
    out, t = [], int(t0_ns)
    for i, (label, ms) in enumerate(phases):
        d = int(round(ms * 1e6))
        out.append(TaskRecord(i, label, stream, t, t + d))
        t += d
    return out


def ring_timeline(tl: dict) -> List[TaskRecord]:
    """Timeline of a ring-of-sections pass (RingOfSections.run's event times,
    ms from the first load): section loads on "h2d", layer computes on
    "compute" -- the streams of ring_offload.cpp:52-106."""
    out = []
    for i, (s, e) in enumerate(zip(tl["load_start"], tl["load_end"])):
        out.append(TaskRecord(len(out), f"load[{i}]", "h2d", int(s * 1e6), int(e * 1e6)))
    for i, (s, e) in enumerate(zip(tl["compute_start"], tl["compute_end"])):
        out.append(TaskRecord(len(out), f"compute[{i}]", "compute", int(s * 1e6), int(e * 1e6)))
    return out
