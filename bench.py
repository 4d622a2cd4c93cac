"""MoE-layer benchmark (BASELINE.json metric: MoE-layer tokens/sec at 1/2/4/8
B200 and % of roofline).

A step = one forward + backward of the MoE layer (gate GEMM, routing,
dispatch, EP all-to-all, expert FFN, all-to-all back, combine, and the
backward of all of it incl. weight gradients) over T tokens per GPU of
synthetic SplitMix64 data.  Workload = config c2 (BASELINE.json configs[1]):
Switch top-1, E = 64, d = 1024, d_ff = 4096, T = 65536 tokens/GPU, bf16,
experts sharded over the N GPUs (weak scaling).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c2]
    torchrun --nproc-per-node N bench.py --gpus N ...

--impl reference times the reference's CPU implementation of the path on the
host cores: the reference has no MoE-layer arithmetic, so this is the CPU
oracle restatement (oracle/, kind "port") on a bounded token sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer tokens/sec at 1/2/4/8 B200; % of HBM/tensor/NVLink roofline"

CONFIGS = {
    "c1": dict(E=8, k=2, d=512, dff=2048, T=4096, cf=1.25, dtype="f32",
               desc="c1: E=8 top-2 MoE FFN layer, d=512, d_ff=2048, T=4096, cf=1.25, fp32 fwd+bwd"),
    "c2": dict(E=64, k=1, d=1024, dff=4096, T=65536, cf=1.25, dtype="bf16",
               desc="c2: Switch top-1 MoE layer fwd+bwd, E=64, d=1024, d_ff=4096 (4d), "
                    "T=65536 tokens/GPU, cf=1.25, bf16, experts sharded E/N per GPU"),
    "c3": dict(E=32, k=2, d=1024, dff=4096, T=65536, cf=1.25, dtype="bf16", skew=1.2,
               desc="c3: E=32 top-2, gate bias calibrated so the top-1 choice follows "
                    "gen_trace's Zipf(s=1.2) expert distribution (workload.cpp:19-53), capacity "
                    "drops, d=1024, d_ff=4096, T=65536/GPU, bf16 fwd+bwd"),
    "c4": dict(E=64, k=2, d=4096, dff=16384, T=16384, cf=1.25, dtype="bf16", layers=2,
               desc="c4: GPT-MoE block stack of 2 MoE layers d=4096, d_ff=16384, E=64 top-2, "
                    "T=16384/GPU, bf16 fwd+bwd; the layers' replicated gate gradients reduced by "
                    "fused gradient buckets (moe_grad_buckets) at N>1"),
}


def zipf_gate_bias(E, skew, sigma=1.0 / 3.0, n=200000, iters=80, seed=2205):
    """Gate bias b such that argmax_e(z_e + b_e), z_e ~ N(0, sigma^2) i.i.d. (the
    gate logits x.wg^T of the synthetic init: x ~ U(-1,1), wg ~ U(-1/sqrt d,
    1/sqrt d) give sigma = 1/3 for any d), picks expert e with probability
    p_e = (e+1)^-skew / H -- the Zipf CDF gen_trace draws each token from
    (workload.cpp:19-53).  Fixed-point iteration on a seeded Monte-Carlo sample
    (deterministic)."""
    import numpy as np
    p = np.array([(e + 1.0) ** -skew for e in range(E)])
    p /= p.sum()
    z = np.random.default_rng(seed).standard_normal((n, E)).astype(np.float32) * np.float32(sigma)
    b = (sigma * np.log(p)).astype(np.float32)
    for _ in range(iters):
        q = np.bincount(np.argmax(z + b, axis=1), minlength=E) / n
        b = b + np.float32(0.5 * sigma) * np.log(p / np.maximum(q, 0.5 / n)).astype(np.float32)
        b -= b.max()
    return [float(v) for v in b]


def gate_bias_for(cfg):
    return zipf_gate_bias(cfg["E"], cfg["skew"]) if cfg.get("skew") else None


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
         "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        for key in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained", "sm_max_mhz"):
            if key in m:
                p[key] = float(m[key])
        p["source"] = "measured (MEASURED_PEAKS.json)"
    return p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ CPU arm --
def cpu_oracle_tokens_per_s(cfg, tokens, seed=2205, repeats=1):
    """Oracle fwd+bwd of the layer on `tokens` tokens (all host threads)."""
    import numpy as np

    import oracle
    E, k, d, dff, cf = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["cf"]
    bf16 = cfg["dtype"] == "bf16"
    t = oracle.make_layer_tensors(seed, tokens, d, dff, E, bf16)
    bg = gate_bias_for(cfg)
    bg = None if bg is None else np.asarray(bg, np.float32)
    C = int(np.ceil(k * cf * tokens / E))
    best = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        fwd = oracle.moe_forward(t["x"], t["wg"], bg, t["w1"], t["b1"], t["w2"], t["b2"], k, C, bf16)
        fwd["logits_used"] = fwd["logits"]
        oracle.moe_backward(t["x"], t["wg"], bg, t["w1"], t["b1"], t["w2"], t["b2"], k, C, bf16,
                            fwd, t["dy"], 0.01)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return tokens / best, best


def cpu_sample_tokens(cfg):
    # ~10-30 s of host work: per-token oracle cost ~ 16 * k * d * dff flops (fp64)
    per_token = 16.0 * cfg["k"] * cfg["d"] * cfg["dff"]
    return int(max(64, min(cfg["T"], 1.0e11 / per_token)) // 64 * 64)


def run_reference_arm(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.set_threads(len(os.sched_getaffinity(0)))  # all host cores, also under torchrun
    n = cpu_sample_tokens(cfg) // 4 if args.steps > 1 else cpu_sample_tokens(cfg)
    n = max(64, n // 64 * 64)
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_oracle_tokens_per_s(cfg, 64)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_oracle_tokens_per_s(cfg, n)
        times.append(dt)
    value = n * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64-accumulate",
        "data": "synthetic (SplitMix64-seeded, rng.hpp)",
        "config": {"workload": cfg["desc"], "sample_tokens_per_step": n},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": oracle.num_threads(),
                         "kind": "port",
                         "sample": f"{n} tokens of {cfg['desc'].split(':')[0]} per step "
                                   "(oracle/moe_oracle.c fwd+bwd; the reference itself has no "
                                   "MoE-layer arithmetic, SPEC.md:15,153,156)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


# The JSON line is the only thing on stdout: native libraries (NCCL's version
# banner, CUDA) print to fd 1, so fd 1 is pointed at stderr for the run and the
# line goes to the saved original stdout.
_JSON_FD = None


def emit(line):
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def _redirect_stdout():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


ALL_CPUS = os.sched_getaffinity(0)


def bind_to_gpu_numa(local):
    """Pin this rank to the CPU cores NVML reports as local to its GPU, so the
    pinned host buffers of the host-buffer (e2e) path are first-touched on the
    GPU's NUMA node and DMA does not cross the socket interconnect."""
    try:
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = int(vis.split(",")[local]) if vis else local
        h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


# ------------------------------------------------------ reference metrics --
def ring_predicted(layers, slots, section_bytes, compute_ns, bw, lat_ns):
    """The reference's ring model (ring_offload.cpp:52-106 on the FIFO streams
    of sim_engine.cpp; transfer time topology.cpp:73-84) for the same plan,
    fed with the measured per-layer compute: predicted makespan / stall."""
    K = min(slots, layers)
    c = lat_ns + -(-section_bytes * 10**9 // int(bw))
    load_end = [0] * layers
    h2d = comp = total = 0
    for i in range(K):
        h2d += c
        load_end[i] = h2d
    end = 0
    for i in range(layers):
        s0 = max(load_end[i], comp)
        comp = s0 + compute_ns[i]
        total += compute_ns[i]
        if i + K < layers:
            h2d = max(h2d, comp) + c
            load_end[i + K] = h2d
    end = max(comp, max(load_end))
    return {"makespan_ms": end / 1e6, "stall_ms": (end - total) / 1e6}


def ring_leg(args, dev, layers=4, slots=2, tokens=131072):
    """Config c5 (ring-of-sections inference) reduced to N=4 layers so the
    pinned sections (2.15 GB each) stay within the bench's time budget; the
    reference's infer-sim metrics (report.cpp:172-187) measured on the CUDA-
    event timeline beside the reference model's prediction for the same plan."""
    import torch

    from paper_2205_10034_b200 import MoEConfig, MoELayer
    from paper_2205_10034_b200.ring import RingOfSections
    t0 = time.time()
    cfg = MoEConfig(8, 2, 4096, 16384, 1.25, tokens, torch.bfloat16)
    layer = MoELayer(cfg, device=dev)
    ring = RingOfSections(layer, layers, slots, seed=5)
    x = layer.make_input(3)
    ring.run(x)
    torch.cuda.synchronize()
    runs = []
    for _ in range(3):
        _, tl = ring.run(x)
        torch.cuda.synchronize()
        runs.append(tl)
    tl = sorted(runs, key=lambda r: r["makespan_ms"])[1]
    sec = tl["section_bytes"]
    loads = [e - s for s, e in zip(tl["load_start"], tl["load_end"])]
    comp_ns = [int(1e6 * (e - s)) for s, e in zip(tl["compute_start"], tl["compute_end"])]
    load_ms = statistics.median(loads)
    out = {
        "config": f"c5 reduced: {layers} layers (of 12), K={tl['slots']} slots, E=8 top-2, "
                  f"d=4096, d_ff=16384, bf16, {tokens} tokens per pass, sections in pinned host "
                  "memory",
        "makespan_ms": tl["makespan_ms"], "compute_total_ms": tl["compute_total_ms"],
        "stall_ms": tl["makespan_ms"] - tl["compute_total_ms"],
        "peak_gpu_bytes": tl["peak_gpu_bytes"], "baseline_gpu_bytes": tl["baseline_gpu_bytes"],
        "memory_reduction": 1.0 - tl["peak_gpu_bytes"] / tl["baseline_gpu_bytes"],
        "tokens_per_s": tokens / (tl["makespan_ms"] / 1e3),
        "section_bytes": sec, "h2d_gbs": sec / load_ms / 1e6,
        "predicted_ref_default_link": ring_predicted(layers, slots, sec, comp_ns, 25e9, 2000),
        "predicted_measured_link": ring_predicted(layers, slots, sec, comp_ns,
                                                  sec / load_ms * 1e3, 2000),
        "note": "predicted_* = the reference's simulate() on this plan with the measured "
                "compute times and PCIe at the reference default (25 GB/s, 2 us; "
                "scenario.cpp:59) or the measured H2D rate",
        "setup_s": time.time() - t0,
    }
    ring.close()
    del ring, layer, x
    torch.cuda.empty_cache()
    return out


def a2a_fusion_leg(ep, ws, rank, E, Cs, d, iters=10):
    """Fusion communication (§4.2, lower_slice_transfer collectives.cpp:
    250-267): the c-config's expert slices (Cs rows x d bf16 each, E/N per peer)
    sent as ONE message per peer vs one per expert slice; device time, max over
    ranks (report.cpp:240-252 metric names)."""
    import torch
    import torch.distributed as dist
    El = max(1, E // ws)
    slice_bytes = Cs * d * 2
    per_peer = El * slice_bytes
    send = torch.empty(ws * per_peer, dtype=torch.uint8, device="cuda").random_(0, 255)
    recv = torch.empty_like(send)
    stream = torch.cuda.current_stream()
    res = {}
    for fused in (True, False):
        for _ in range(2):
            ep.alltoall_packed(send, recv, per_peer, El, fused)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            ep.alltoall_packed(send, recv, per_peer, El, fused)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        res["fused_ms" if fused else "unfused_ms"] = float(ms.item())
    out_bytes = per_peer * (ws - 1)
    del send, recv
    torch.cuda.empty_cache()
    return {"slices_per_peer": El, "slice_bytes": slice_bytes, "bytes_out_per_gpu": out_bytes,
            "fused_ms": res["fused_ms"], "unfused_ms": res["unfused_ms"],
            "fused_gbs": out_bytes / res["fused_ms"] / 1e6,
            "unfused_gbs": out_bytes / res["unfused_ms"] / 1e6,
            "speedup": res["unfused_ms"] / res["fused_ms"],
            "api": "moe_alltoall_packed (NCCL over NVLink)"}


# ------------------------------------------------------------------ GPU arm --
def main():
    _redirect_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--tokens", type=int, default=0, help="override T (tokens per GPU)")
    ap.add_argument("--layers", type=int, default=0,
                    help="override the MoE layers per step (block stack; c4 default 2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ring", action="store_true",
                    help="skip the reduced c5 ring-of-sections leg (N=1 only)")
    ap.add_argument("--timeline", default="",
                    help="write the profiled step's phase timeline as trace-event JSON here")
    ap.add_argument("--placement", default="round_robin", choices=["contiguous", "round_robin"],
                    help="expert placement over the N GPUs (include/moe_b200.h); round-robin "
                         "spreads a skewed gate's hot experts over the ranks (c3 N=4: 2.3x), "
                         "neutral for uniform routing (c2)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="EP token exchange for N>1: NVLink peer stores (p2p) or NCCL all-to-all")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.tokens:
        cfg["T"] = args.tokens
    if args.layers:
        cfg["layers"] = args.layers
    L = int(cfg.get("layers", 1))
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch
    import torch.distributed as dist

    from paper_2205_10034_b200 import EPGroup, MoEConfig, MoELayer, kernel_launch_count
    from paper_2205_10034_b200.layer import T_DY

    ws, rank, local = dist_env()
    assert args.gpus == ws or ws == 1, "--gpus must match WORLD_SIZE"
    numa_cpus = bind_to_gpu_numa(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ep = None
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
        ep = EPGroup(ws, rank)
    dtype = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    E, k, d, dff, T, cf = cfg["E"], cfg["k"], cfg["d"], cfg["dff"], cfg["T"], cfg["cf"]
    mcfg = MoEConfig(E, k, d, dff, cf, T, dtype, gate_bias=bool(cfg.get("skew")),
                     exchange=args.exchange, placement=args.placement)
    if L > 1:
        from paper_2205_10034_b200.stack import MoEStack
        model = MoEStack(mcfg, L, ep=ep, device=dev)
        layer = model.layers[0]
    else:
        model = layer = MoELayer(mcfg, ep=ep, device=dev)
    gb = gate_bias_for(cfg)
    gb = None if gb is None else torch.tensor(gb, dtype=torch.float32, device=dev)
    model.init_params(1234, gate_bias=gb)
    x = model.make_input(1234)
    dy = model.make_input(1234, T_DY)
    stream = torch.cuda.current_stream()

    def step():
        model.forward(x)
        model.backward(dy, d_aux=0.01)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-timed region: exactly K steps, inputs resident in HBM ----
    sampler = ClockSampler(local)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    sampler.start()
    n0 = kernel_launch_count()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    barrier()
    launches = kernel_launch_count() - n0
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)

    # ---- separate profiled pass: per-phase CUDA events on the launch stream ----
    barrier()  # ranks leave the clock sampler at different times: re-align first
    model.set_profiling(True)
    phase_tot = {}
    # K steps back to back without a host sync (the host stays ahead of the
    # GPU, so no phase carries a host-enqueue gap); the last step's per-phase
    # events stand for every step
    for _ in range(args.steps):
        model.forward(x)
        model.backward(dy, d_aux=0.01)
    fwd_ph = model.phase_list("fwd")
    bwd_ph = model.phase_list("bwd")
    for n, v in fwd_ph:
        phase_tot["fwd." + n] = phase_tot.get("fwd." + n, 0.0) + v * args.steps
    for n, v in bwd_ph:
        phase_tot["bwd." + n] = phase_tot.get("bwd." + n, 0.0) + v * args.steps
    model.set_profiling(False)
    if args.timeline and rank == 0:
        # the last profiled step as the reference's trace-event JSON
        # (trace_export.cpp:28-58; TaskRecord per phase on the launch stream)
        from paper_2205_10034_b200 import moesim
        tasks = moesim.layer_step_timeline([("fwd." + n, v) for n, v in fwd_ph] +
                                           [("bwd." + n, v) for n, v in bwd_ph],
                                           stream=f"rank{rank}.compute")
        moesim.export_trace(tasks, args.timeline)
    barrier()
    t_ms = torch.tensor([ms], device=dev)
    if ws > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms = float(t_ms.item())
    ms_step = ms / args.steps
    value = ws * T * args.steps / (ms / 1000.0)

    # routing statistics of the last step
    _, rout = layer.forward(x, routing=True)
    torch.cuda.synchronize()
    kept_local = int(rout["kept"].sum().item())
    count1 = rout["count1"].float()
    imb = float(count1.max().item() / max(count1.mean().item(), 1e-9))
    drop = 1.0 - kept_local / float(T * k)
    imb_ref = None
    if cfg.get("skew"):
        # the reference's statistic of its own skewed trace (workload.cpp:19-66)
        # through this package's drop-in gen_trace / imbalance_ratio (golden-pinned)
        from paper_2205_10034_b200 import moesim
        imb_ref = moesim.imbalance_ratio(moesim.gen_trace(7, 1, 1, E, T, cfg["skew"]))

    # ---- roofline of the dominant kernel (expert grouped GEMMs, tcgen05) ----
    pk = peaks()
    gemm_phases = ["fwd.ffn1", "fwd.ffn2", "bwd.dgrad_ffn2", "bwd.dgrad_ffn1", "bwd.wgrad_w1",
                   "bwd.wgrad_w2"]
    gemm_ms = sum(phase_tot.get(p, 0.0) for p in gemm_phases) / args.steps
    # algorithmic flops per step on this GPU: rows the local experts processed
    kept_t = torch.tensor([kept_local], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(kept_t)
    rows_local = float(kept_t.item()) / ws  # EP: on average each GPU computes T*k kept rows
    flops_step = L * 6 * 2.0 * rows_local * d * dff
    achieved_tf = flops_step / (gemm_ms / 1000.0) / 1e12 if gemm_ms > 0 else None
    prof_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    traffic = None
    if os.path.exists(prof_path):
        with open(prof_path) as f:
            traffic = json.load(f).get(args.config, {}).get("dram_bytes_per_launch")
    # Timed region of a few hundred ms at (near) max SM clock -> the burst
    # peak is the honest denominator; a long, clock-capped run -> sustained.
    burst = (clocks.get("sm_mhz") or 0) >= 0.95 * (clocks.get("sm_max_mhz") or 1e9) and ms < 2000
    if dtype == torch.bfloat16:
        peak = pk["bf16_tflops"] if burst else pk["bf16_tflops_sustained"]
        kname, bound = ("tc_gemm_kernel (6 expert GEMMs/step: ffn1, ffn2, 2x dgrad, 2x wgrad)",
                        "tensor")
        psrc = pk["source"] + (", burst (timed region at max SM clock)" if burst else ", sustained")
    elif d % 128 == 0 and dff % 128 == 0 and os.environ.get("MOE_F32_GEMM") != "simt":
        # c1: fp32 expert GEMMs as split-bf16 tcgen05 GEMMs (f32split.cu): six
        # bf16 plane products per fp32 product, so the fp32 ceiling is 1/6 of bf16
        peak = (pk["bf16_tflops"] if burst else pk["bf16_tflops_sustained"]) / 6.0
        kname, bound = ("tc_gemm_kernel split-fp32 (6 expert GEMMs/step as 6 bf16 plane products, "
                        "K chunks of 512 summed in fp32; incl. split / finish kernels)", "tensor")
        psrc = pk["source"] + (", burst" if burst else ", sustained") + " bf16 / 6"
    else:  # fp32 SIMT GEMMs
        props = torch.cuda.get_device_properties(dev)
        peak = props.multi_processor_count * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        kname, bound = "simt_gemm_kernel (6 expert GEMMs/step, fp32 FFMA)", "fp32"
        psrc = "nominal FP32 FFMA: SMs x 128 lanes x 2 x max SM clock"
    if traffic is not None:  # ncu: DRAM bytes of the six GEMM launches of one step
        traffic_step, traffic = traffic, traffic / 6.0
    else:
        traffic_step = None
    roof = {"kernel": kname, "bound": bound, "achieved": achieved_tf, "peak": peak,
            "unit": "TFLOP/s", "frac": (achieved_tf / peak) if achieved_tf else None,
            "traffic": traffic, "traffic_note": "mean DRAM bytes per GEMM launch (ncu --set "
            "full, profiles/ncu_summary.json); traffic_per_step = the six launches",
            "traffic_per_step": traffic_step, "peak_source": psrc,
            "peak_burst": pk["bf16_tflops"] if dtype == torch.bfloat16 else None,
            "peak_sustained": pk["bf16_tflops_sustained"] if dtype == torch.bfloat16 else None,
            "frac_vs_sustained": (achieved_tf / pk["bf16_tflops_sustained"])
            if achieved_tf and dtype == torch.bfloat16 else None,
            "flops_per_step": flops_step, "gemm_ms_per_step": gemm_ms,
            "gemm_share_of_step": gemm_ms / ms_step if ms_step else None}
    # per-GEMM view: each of the six carries 2 * rows * d * d_ff flops; its
    # algorithmic HBM bytes are its operands + outputs once:
    # activations R x {d, d_ff}, weights E_local x d x d_ff, fp32 dW
    es = 2 if dtype == torch.bfloat16 else 4
    R, W = rows_local, (E // ws) * d * dff
    gbytes = {"ffn1": es * (R * d + W + 2 * R * dff),          # X, W1 -> A, gelu'(h)
              "ffn2": es * (R * dff + W + R * d),              # A, W2 -> Y
              "dgrad_ffn2": es * (R * d + W + 2 * R * dff),    # dY, W2, gelu'(h) -> dH
              "dgrad_ffn1": es * (R * dff + W + R * d),        # dH, W1 -> dX
              "wgrad_w1": es * (R * d + R * dff) + 4 * W,      # X, dH -> dW1 (fp32)
              "wgrad_w2": es * (R * dff + R * d) + 4 * W}      # A, dY -> dW2 (fp32)
    per = []
    for name in ("ffn1", "ffn2", "dgrad_ffn2", "dgrad_ffn1", "wgrad_w1", "wgrad_w2"):
        ms_k = sum(v for n, v in phase_tot.items() if n.split(".", 1)[-1] == name) / args.steps
        if ms_k > 0:
            tf = L * 2.0 * rows_local * d * dff / (ms_k / 1000.0) / 1e12
            gbs = L * gbytes[name] / (ms_k / 1000.0) / 1e9
            per.append({"gemm": name, "ms": ms_k, "tflops": tf, "frac": tf / peak,
                        "hbm_GBps": gbs, "hbm_frac": gbs / pk["hbm_gbs"]})
    roof["per_gemm"] = per
    if dtype == torch.bfloat16 and rank == 0:
        # library reference: cuBLAS on the dense equivalent of each expert GEMM
        # shape (all kept rows as one matrix, bf16 in, fp32 accumulate, bf16
        # out, no epilogue) on the same GPU -- what a plain GEMM reaches here
        R_ = int(rows_local) // 128 * 128
        shapes = {"ffn1 (R x d -> d_ff)": (R_, d, dff), "ffn2 (R x d_ff -> d)": (R_, dff, d)}
        cub = {}
        for nm, (mm, kk, nn) in shapes.items():
            a_ = torch.randn(mm, kk, device=dev, dtype=torch.bfloat16)
            b_ = torch.randn(kk, nn, device=dev, dtype=torch.bfloat16)
            for _ in range(3):
                torch.matmul(a_, b_)
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0_.record()
            for _ in range(10):
                torch.matmul(a_, b_)
            e1_.record()
            torch.cuda.synchronize()
            t_ = e0_.elapsed_time(e1_) / 10
            cub[nm] = {"ms": t_, "tflops": 2.0 * mm * kk * nn / (t_ / 1e3) / 1e12}
            del a_, b_
        roof["cublas_dense_equivalent"] = cub

    # ---- HBM roofline of the memory-bound kernels (gating, dispatch, combine
    # and their backward): algorithmic bytes = each operand read once + each
    # output written once, R = kept rows of this rank's tokens,
    # time = the phase's CUDA events (includes its launch gap).  At N > 1 the
    # dispatch / combine-backward phases also carry the NVLink exchange and
    # are reported under "nvlink" instead.
    Rk = float(kept_local)
    Ep = (E + 63) // 64 * 64 if dtype == torch.bfloat16 else E
    hbytes = {
        "gate_gemm": T * d * es + T * E * 4,                          # x -> logits (fp32)
        "route": T * E * 4 + T * k * 13,                               # logits -> e, g, pos, keep
        "dispatch": T * d * es + Rk * d * es,                          # x -> expert-major rows
        "combine": Rk * d * es + T * d * es,                           # Y rows -> y
        "combine_bwd": T * d * es + 2 * Rk * d * es,                   # dy, Y -> dY rows
        "route_bwd": T * E * 4 + T * Ep * es,                          # logits -> dlogits
        "bias_grads": Rk * d * es,                                     # dY -> db2
        "gate_wgrad": T * d * es + T * Ep * es,                        # x, dlogits -> dWg
        "gate_dgrad_gather_dx": T * Ep * es + Rk * d * es + T * d * es,  # dlogits, dXe -> dx
    }
    if ws > 1:  # the P2P combine backward pushes its rows over NVLink
        hbytes.pop("combine_bwd")
    hbm = []
    for name, nbytes in hbytes.items():
        ms_k = sum(v for n, v in phase_tot.items() if n.split(".", 1)[-1] == name) / args.steps
        if ms_k > 0:
            gbs = L * nbytes / (ms_k / 1000.0) / 1e9
            hbm.append({"kernel": name, "us": 1000.0 * ms_k, "bytes": L * nbytes, "GBps": gbs,
                        "frac": gbs / pk["hbm_gbs"]})
    roof["hbm_kernels"] = hbm

    # ---- end to end through the host-buffer API (H2D + step + D2H) ----
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        dyh = dy.cpu().pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        dxh = torch.empty_like(xh).pin_memory()
        if L == 1:
            def host_step():
                layer.train_step_host(xh, dyh, yh, dxh, d_aux=0.01, deferred=True)
        else:  # block stack: H2D, stack fwd + bwd, D2H on the stream
            def host_step():
                xd = xh.to(dev, non_blocking=True)
                dyd = dyh.to(dev, non_blocking=True)
                yh.copy_(model.forward(xd), non_blocking=True)
                dxh.copy_(model.backward(dyd, d_aux=0.01), non_blocking=True)
        host_step()
        if L == 1:
            layer.host_sync()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            host_step()
        if L == 1:
            layer.host_sync()  # the last step's y / dx have landed in host memory
        ev1.record(stream)
        barrier()
        e_ms = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
        if ws > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms = float(e_ms.item())
        nbytes = T * d * (2 if dtype == torch.bfloat16 else 4)
        e2e = {"value": ws * T * args.steps / (e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * nbytes, "d2h_bytes_per_step": 2 * nbytes,
               "ms_per_step": e_ms / args.steps,
               "api": ("moe_layer_train_step_host_async x K + moe_layer_host_sync "
                       "(pinned x, dy -> y, dx; every step's copies inside the timed region)")
                      if L == 1 else "MoEStack fwd/bwd with pinned x, dy -> y, dx copies "
                                     "on the stream",
               "host_cpus_bound": numa_cpus}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        os.sched_setaffinity(0, ALL_CPUS)  # the CPU baseline gets every host core
        import oracle
        oracle.set_threads(len(ALL_CPUS))
        n = cpu_sample_tokens(cfg)
        v, dt = cpu_oracle_tokens_per_s(cfg, n)
        cpu = {"value": v, "unit": "tokens/s", "cores": oracle.num_threads(), "kind": "port",
               "sample": f"{n} tokens of the {args.config} layer fwd+bwd ({dt:.1f} s, "
                         "oracle/moe_oracle.c fp64-accumulate, OpenMP)"}

    ring = None
    if rank == 0 and ws == 1 and not args.no_ring and dtype == torch.bfloat16:
        ring = ring_leg(args, dev)
    a2a_fusion = a2a_fusion_leg(ep, ws, rank, E, model.capacity, d) if ws > 1 else None

    a2a_ms = sum(v for n, v in phase_tot.items() if ".a2a" in n) / args.steps
    nvlink = None
    if ws > 1:
        # token rows that cross NVLink per exchange per GPU: kept rows owned by
        # other ranks (uniform routing: (P-1)/P of them), d * 2 bytes each
        row_bytes = d * (2 if dtype == torch.bfloat16 else 4)
        xbytes = L * kept_local * row_bytes * (ws - 1) / ws  # summed over the stack's layers
        ph = {n: v / args.steps for n, v in phase_tot.items()}
        if args.exchange == "p2p":
            ex = {"dispatch": ph.get("fwd.a2a_counts", 0) + ph.get("fwd.dispatch_p2p", 0) +
                  ph.get("fwd.a2a_dispatch", 0),
                  "combine": ph.get("fwd.a2a_combine", 0),
                  "dy": ph.get("bwd.combine_bwd", 0) + ph.get("bwd.a2a_dy", 0),
                  "dx": ph.get("bwd.a2a_dx", 0)}
        else:
            ex = {"dispatch": ph.get("fwd.a2a_dispatch", 0), "combine": ph.get("fwd.a2a_combine", 0),
                  "dy": ph.get("bwd.a2a_dy", 0), "dx": ph.get("bwd.a2a_dx", 0)}
        if args.exchange == "p2p" and dtype == torch.bfloat16:
            # Y and dX return inside the ffn2 / dgrad_ffn1 epilogues (overlapped with
            # the MMAs): only the dispatch and dY exchanges are exposed transfers
            exposed = {n: ex[n] for n in ("dispatch", "dy")}
            moved = 2 * xbytes
        else:
            exposed = ex
            moved = 4 * xbytes
        ex_ms = sum(exposed.values())
        ach = moved / (ex_ms / 1000.0) / 1e9 if ex_ms > 0 else None
        nvlink = {"bound": "nvlink", "unit": "GB/s", "achieved": ach,
                  "peak": 900.0, "peak_source": "NVLink 5 nominal per direction per GPU; "
                  "770 = measured peer-copy guide number (B200_PROFILING.md)",
                  "frac": ach / 900.0 if ach else None,
                  "frac_vs_770": ach / 770.0 if ach else None,
                  "bytes_per_exchange_per_gpu": xbytes, "exchanges_per_step": 4,
                  "exposed_exchange_ms": exposed, "all_exchange_phase_ms": ex,
                  "note": ("dispatch / dY exchanges fused into the dispatch and combine-backward "
                           "kernels (phase time incl. the count all-gather and peer skew); Y and "
                           "dX returns fused into GEMM epilogues, not exposed")
                  if args.exchange == "p2p" else "ncclAlltoAll of capacity-padded buffers"}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (SplitMix64-seeded x, dy and weights; rng.hpp substreams)",
        "config": {"workload": cfg["desc"], "tokens_per_gpu": T, "experts": E, "top_k": k,
                   "d_model": d, "d_ff": dff, "capacity_factor": cf,
                   "capacity": model.capacity, "experts_per_gpu": E // ws, "layers": L,
                   "parallelism": f"ep{ws}" if ws > 1 else "single",
                   "exchange": args.exchange if ws > 1 else None,
                   "placement": args.placement if ws > 1 else None,
                   "l2": "inputs larger than L2 (x 128 MiB + weights 1 GiB per step), no flush"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks,
        "routing": {"imbalance_ratio": imb, "drop_rate": drop,
                    "gen_trace_imbalance_ratio": imb_ref,
                    "note": "imbalance over top-1 choices (max/mean count1); gen_trace_* = "
                            "imbalance_ratio(gen_trace(7, 1, 1, E, T, skew)) of the reference's "
                            "Zipf generator"
                            if imb_ref else "imbalance over top-1 choices (max/mean count1)"},
        "a2a_ms_per_step": a2a_ms if ws > 1 else 0.0,
        "ring": ring, "a2a_fusion": a2a_fusion,
        "nvlink": nvlink,
        "phases_ms_per_step": {n: v / args.steps for n, v in sorted(phase_tot.items())},
    }
    if rank == 0:
        emit(line)
    if ep is not None:
        model.close()
        ep.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
