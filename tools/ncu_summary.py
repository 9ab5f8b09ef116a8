"""Summarise ncu captures into profiles/ (run here, on the CPU side).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_<name>.md
    python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/r01_launches.md

Full captures (`ncu --set full`): per kernel duration, cycles, DRAM bytes,
achieved HBM GB/s, tensor-pipe activity, occupancy, registers and the top
warp-stall reasons.  Launch lists (`--metrics gpu__time_duration.sum`): time
per kernel family and its share of the step.
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("sm__cycles_elapsed.avg", "cycles", 1),
    ("dram__bytes_read.sum", "DRAM read (B)", 1),
    ("dram__bytes_write.sum", "DRAM write (B)", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %", 1),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc inst %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
    ("launch__registers_per_thread", "regs/thread", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
    ("smsp__inst_executed.sum", "warp instr", 1),
]


_UNIT = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3,
         "ms": 1e6, "s": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "Kibyte": 1024.0, "Mibyte": 1024.0 ** 2}


def _num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def summarize_rep(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    out = [f"# ncu summary of `{path}`", "",
           "| kernel | " + " | ".join(m[1] for m in METRICS) + " | HBM GB/s | top stalls |",
           "|" + "---|" * (len(METRICS) + 3)]
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    for row in rows[2:]:
        if len(row) < len(hdr):
            continue
        name = row[hdr.index("Kernel Name")]
        vals = []
        got = {}
        for key, _label, scale in METRICS:
            v = _num(row[hdr.index(key)]) if key in hdr else None
            if v is not None and key in hdr:
                v *= _UNIT.get(units[hdr.index(key)], 1.0)  # → ns / bytes
            got[key] = v
            vals.append("" if v is None else (f"{v * scale:.2f}" if scale != 1 else f"{v:.0f}"))
        dur_ns = got.get("gpu__time_duration.sum")
        rd = got.get("dram__bytes_read.sum") or 0
        wr = got.get("dram__bytes_write.sum") or 0
        gbs = (rd + wr) / dur_ns if dur_ns else 0.0
        stalls = sorted(((_num(row[i]) or 0, hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for i in stall_cols), reverse=True)[:4]
        st = ", ".join(f"{n} {int(v)}" for v, n in stalls if v)
        out.append(f"| `{name[:70]}` | " + " | ".join(vals) + f" | {gbs:.1f} | {st} |")
    return "\n".join(out) + "\n"


def summarize_launches(path: str) -> str:
    fam = defaultdict(lambda: [0.0, 0])
    total = 0.0
    with open(path) as fh:
        text = fh.read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = _num(r[vi]) or 0.0
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "nsecond"
        unit_scale = _UNIT.get(unit, 1.0) * 1e-3  # → us
        name = r[ki].split("(")[0].replace("void ", "").strip()
        fam[name][0] += v * unit_scale
        fam[name][1] += 1
        total += v * unit_scale
    out = [f"# ncu launch list `{path}` (cold-cache, serialised: compare shares)", "",
           f"total kernel time {total:.1f} us over {sum(c for _, c in fam.values())} launches", "",
           "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (t, c) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
        out.append(f"| `{name[:80]}` | {c} | {t:.1f} | {100 * t / total:.1f}% |")
    return "\n".join(out) + "\n"


# kernel-name substring -> engine task family (first match wins: the
# sepconv names come before "conv_tc_kernel", a substring of "sepconv_tc_kernel")
FAMILY = {"sepconv_kernel": "sepconv", "sepconv_tma_kernel": "sepconv", "sepconv_tc_kernel": "sepconv",
          "sep_rows_kernel": "sepconv", "conv_simt_kernel": "conv", "conv_tc_kernel": "conv",
          "conv_tc_tma": "conv", "conv_tcs_kernel": "conv", "conv_pw_tc_kernel": "conv",
          "conv_direct_kernel": "conv", "pw_tma_kernel": "conv", "conv_gemv_kernel": "conv",
          "spatial_kernel<0": "dwconv", "spatial_kernel<1": "pool", "spatial_rows_kernel<0": "dwconv",
          "spatial_rows_kernel<1": "pool", "pool_rows_kernel": "pool", "global_pool": "gpool", "ew_": "eltwise"}


def traffic_json(path: str) -> dict:
    """Mean DRAM bytes (read + write) per launch, by engine task family."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    acc = defaultdict(list)
    for row in rows[2:]:
        if len(row) < len(hdr):
            continue
        name = row[hdr.index("Kernel Name")]
        fam = next((f for k, f in FAMILY.items() if k in name), None)
        if fam is None:
            continue
        b = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = _num(row[hdr.index(key)]) or 0.0
            b += v * _UNIT.get(units[hdr.index(key)], 1.0)
        acc[fam].append(b)
    return {f: sum(v) / len(v) for f, v in acc.items()}


def main():
    if sys.argv[1] == "--traffic":
        import json
        d = traffic_json(sys.argv[2])
        with open(sys.argv[3], "w") as fh:
            json.dump(d, fh, indent=1)
        print(d)
        return
    if sys.argv[1] == "--launches":
        text = summarize_launches(sys.argv[2])
        dst = sys.argv[3]
    else:
        text = summarize_rep(sys.argv[1])
        dst = sys.argv[2]
    with open(dst, "w") as fh:
        fh.write(text)
    print(text)


if __name__ == "__main__":
    main()
