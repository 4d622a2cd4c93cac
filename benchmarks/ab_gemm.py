"""Interleaved A/B of libmoe_b200.so variants on the GEMM micro-benchmark:
rounds x variants separate processes (ABAB...), min and median per (variant,
GEMM).  python benchmarks/ab_gemm.py --variants base pf --rounds 4 [--only ...]"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--variants", nargs="+", required=True)
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--only", default="")
ap.add_argument("--reps", type=int, default=15)
a = ap.parse_args()
here = os.path.dirname(os.path.abspath(__file__))
res = {}
for r in range(a.rounds):
    for v in a.variants:
        env = dict(os.environ, MOE_B200_LIB=os.path.join(here, "..", "exp", v, "libmoe_b200.so"))
        out = subprocess.run([sys.executable, os.path.join(here, "gemm_sweep.py"), "--json",
                              "--reps", str(a.reps), "--only", a.only], env=env,
                             capture_output=True, text=True, timeout=150)
        for line in out.stdout.splitlines():
            d = json.loads(line)
            res.setdefault(d["name"], {}).setdefault(v, []).append(d["us"])
for name, vs in res.items():
    print(name)
    for v, ts in vs.items():
        print(f"   {v:10s} min {min(ts):7.1f}  med {statistics.median(ts):7.1f}  {[round(t) for t in ts]}")
