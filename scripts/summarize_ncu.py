"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and one `--set full`
capture of the numeric kernel into profiles/<tag>_ncu_summary.md (+ .json).

    python scripts/summarize_ncu.py <tag> gpurun_out/launches_<tag>.csv gpurun_out/prof_numeric_<tag>.ncu-rep
"""

from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
STEP_KERNELS = ("k_decode_rows", "k_row_ptr", "k_gather_u32", "k_cols_rowptr", "k_sym_", "k_combine", "k_inv_counts", "k_iota",
                "k_numeric", "k_block_stats", "k_flags", "k_compact", "DeviceRadixSort", "DeviceScan",
                "Onesweep", "Histogram", "ExclusiveSum", "cub::", "vectorized_elementwise",
                "elementwise")
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def short(name: str) -> str:
    m = re.search(r"(k_\w+|Device\w+Kernel\w*|\w*Onesweep\w*|\w+Kernel)", name)
    base = m.group(1) if m else name[:60]
    cfg = re.search(r"DmmaCfg<\(int\)(\d+)", name)
    return f"{base}<bs{cfg.group(1)}>" if cfg else base


def launches(path: Path):
    text = path.read_text()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        nm = r["Kernel Name"]
        if not any(k in nm for k in STEP_KERNELS):
            continue
        s = short(nm)
        per[s][0] += 1
        per[s][1] += float(r["Metric Value"].replace(",", "")) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
    tot = sum(v[1] for v in per.values())
    return {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 4)} for k, v in
            sorted(per.items(), key=lambda kv: -kv[1][1])}, tot


def full(path: Path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for vals in rows[2:]:
        name = short(vals[hdr.index("Kernel Name")])
        d = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{vals[i]} {units[i]}".strip()
        res[name] = d
    return res


def main():
    tag, lpath, fpath = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3])
    per, tot = launches(lpath)
    fm = full(fpath)
    outj = {"tag": tag, "launch_list": per, "launch_total_us": round(tot, 1), "numeric_full": fm}
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    (prof / f"{tag}_ncu_summary.json").write_text(json.dumps(outj, indent=1))
    lines = [f"# ncu summary {tag}", "", "Launch list (cold-cache, serialised; compare SHARES):", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in per.items():
        lines.append(f"| {k} | {v['launches']} | {v['us']} | {v['share']:.3f} |")
    for k, d in fm.items():
        lines += ["", f"`--set full` capture: {k}", "", "| metric | value |", "|---|---|"]
        lines += [f"| {m} | {v} |" for m, v in d.items()]
    (prof / f"{tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
