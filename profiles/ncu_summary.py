"""Summarise ncu captures into profiles/: per-kernel table (markdown) and the
JSON that bench.py reads for roofline.traffic.

    python profiles/ncu_summary.py --rep gpurun_out/prof.ncu-rep --tag r01 \
        [--launches gpurun_out/launches.csv] [--config c2]

--rep      an `ncu --set full` report (read with `ncu -i ... --page raw --csv`)
--launches a `--metrics gpu__time_duration.sum --csv` launch list of bench.py
Writes profiles/<tag>_ncu.md and merges {config: {...}} into
profiles/ncu_summary.json (expert-GEMM DRAM bytes per step = the sum over the
six tc_gemm launches of one step, i.e. per launch of the roofline's kernel
group).
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import OrderedDict

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = OrderedDict([
    ("gpu__time_duration.sum", "time"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
])
ROLE = {
    "<256, 0, 0, 0, 1, 0, 2, 0>": "ffn1 (GeLU + gelu' epilogue)",
    "<256, 0, 0, 0, 0, 0, 2, 0>": "ffn2",
    "<256, 0, 1, 0, 2, 0, 2, 0>": "dgrad ffn2 (x gelu', fused db1)",
    "<256, 0, 1, 0, 0, 0, 2, 0>": "dgrad ffn1",
    "<256, 1, 1, 1, 0, 1, 2, 0>": "wgrad (fp32 dW)",
    "<256, 0, 1, 0, 4, 0, 2, 0>": "gate dgrad + gather dx",
    "<64, 1, 1, 1, 3, 1, 1, 0>": "gate wgrad (atomic)",
    "<64, 1, 1, 1, 0, 1, 1, 0>": "gate wgrad (split-K partials)",
    "<64, 0, 0, 0, 0, 1, 1, 0>": "gate logits",
    "<256, 0, 0, 0, 0, 0, 2, 1>": "ffn2 + remote Y return (EP)",
    "<256, 0, 1, 0, 0, 0, 2, 1>": "dgrad ffn1 + remote dX return (EP)",
}


def short(name):
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"^void ", "", n)
    n = n.replace("moe::tc::", "").replace("moe::<unnamed>::", "")
    m = re.search(r"<[^>]*>$", n)
    return n, (ROLE.get(m.group(0), "") if m else "")


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def fnum(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    lines = [f"# ncu summary `{a.tag}` (config {a.config})", "",
             "`ncu --set full --clock-control none` (cold cache, serialised replay): kernel shares,",
             "not absolute step times. DRAM bytes per launch.", ""]
    gemm_bytes = []
    for rep in a.rep:
        hdr, units, data = read_raw(rep)
        ki = hdr.index("Kernel Name")
        cols = [(hdr.index(k), lbl, units[hdr.index(k)]) for k, lbl in METRICS.items() if k in hdr]
        lines.append(f"## `{os.path.basename(rep)}`")
        lines.append("")
        lines.append("| kernel | role | " + " | ".join(f"{lbl} ({u})" if u and u != "%" else lbl
                                                      for _, lbl, u in cols) + " |")
        lines.append("|---|---|" + "---|" * len(cols))
        for r in data:
            n, role = short(r[ki])
            vals = []
            for i, _, _ in cols:
                v = fnum(r[i])
                vals.append("" if v is None else (f"{v:.3g}" if v < 100 else f"{v:.0f}"))
            lines.append(f"| `{n}` | {role} | " + " | ".join(vals) + " |")
            if "tc_gemm_kernel<256" in n and "4, 0, 2" not in n:
                rd = fnum(r[hdr.index("dram__bytes_read.sum")])
                wr = fnum(r[hdr.index("dram__bytes_write.sum")])
                mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
                u = units[hdr.index("dram__bytes_read.sum")]
                gemm_bytes.append((rd + wr) * mult.get(u, 1.0))
        lines.append("")
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        h = rows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
        seq = [(short(r[ki])[0], fnum(r[vi]) * scale.get(r[ui], 1.0)) for r in rows[1:]]
        # our kernels only: drop torch's and the cuBLAS reference GEMMs the
        # bench times after the steps (roofline.cublas_dense_equivalent)
        lib = ("nvjet", "cublas", "cutlass", "sm90_", "sm100_", "at::", "void at::")
        seq = [(n, t) for n, t in seq if not n.startswith(lib) and "at::native" not in n]
        # the last full step: from the last gate-logits GEMM (first launch of
        # a step) on, our kernels only
        starts = [i for i, (n, _) in enumerate(seq) if n.endswith("<64, 0, 0, 0, 0, 1, 1, 0>")]
        segs = [seq[s0:s1] for s0, s1 in zip(starts, starts[1:] + [len(seq)])] or [seq]
        step = max(reversed(segs), key=len)  # the latest complete fwd+bwd step
        step = [(n, t) for n, t in step if not n.startswith("at::") and "at::" not in n[:20]]
        tot = sum(t for _, t in step)
        lines.append(f"## launch list `{os.path.basename(a.launches)}`: last step, {len(step)} launches, "
                     f"{tot:.1f} us of kernel time")
        lines.append("")
        lines.append("| # | kernel | role | us | share of step |")
        lines.append("|---|---|---|---|---|")
        for i, (n, t) in enumerate(step):
            role = ROLE.get(re.search(r"<[^>]*>$", n).group(0), "") if re.search(r"<[^>]*>$", n) else ""
            lines.append(f"| {i} | `{n}` | {role} | {t:.1f} | {100 * t / tot:.1f} % |")
        lines.append("")
    md = os.path.join(HERE, f"{a.tag}_ncu.md")
    with open(md, "w") as f:
        f.write("\n".join(lines) + "\n")
    js = os.path.join(HERE, "ncu_summary.json")
    doc = json.load(open(js)) if os.path.exists(js) else {}
    if gemm_bytes:
        doc[a.config] = {"dram_bytes_per_launch": sum(gemm_bytes), "kernels": len(gemm_bytes),
                         "what": "sum of DRAM read+write bytes of the expert-GEMM launches of one step "
                                 "(ncu --set full, cold cache)",
                         "source": f"profiles/{a.tag}_ncu.md"}
        with open(js, "w") as f:
            json.dump(doc, f, indent=1)
    print(md)


if __name__ == "__main__":
    main()
