"""Summarize ncu output brought back from gpurun into committed profiles/.

    python profiles/summarize.py launches <launch-list.csv> <out.md>
    python profiles/summarize.py full <report.ncu-rep> <out.md> [--traffic-key CONFIG]

`launches`: per-kernel launch count, mean / total device time and share of the
listed time (ncu --metrics gpu__time_duration.sum --clock-control none: cold,
serialised launches — compare shares, not absolutes).
`full`: the roofline-relevant counters of an `ncu --set full` capture; with
--traffic-key the per-launch DRAM bytes are merged into profiles/traffic.json,
which bench.py reads for roofline.traffic.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def short(name: str) -> str:
    return name.replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "").split("(")[0]


def launches(csv_path: str, out_md: str) -> None:
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        agg.setdefault((short(r[ki]), r[gi]), []).append(float(r[vi].replace(",", "")) / 1e3)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# Launch list: `{Path(csv_path).name}`", "",
             "ncu `gpu__time_duration.sum`, `--clock-control none`; cold, serialised launches.", "",
             "| kernel | grid | launches | mean us | total ms | share |", "|---|---|---|---|---|---|"]
    for (k, g), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {g} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / 1e3:.3f} | "
                     f"{100 * sum(v) / total:.1f} % |")
    Path(out_md).write_text("\n".join(lines) + "\n")


def full(rep: str, out_md: str, traffic_key: str | None) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full: `{Path(rep).name}`", ""]
    traffic = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        name = short(d["Kernel Name"])
        lines += [f"## `{name}`", "", "| counter | value |", "|---|---|"]
        for key, label in FULL_METRICS:
            if key in d:
                lines.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
        lines.append("")
        try:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
            wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
            base = name.split("<")[0]
            traffic.setdefault(base, rd + wr)
        except Exception:
            pass
    Path(out_md).write_text("\n".join(lines) + "\n")
    if traffic_key:
        tf = HERE / "traffic.json"
        cur = json.loads(tf.read_text()) if tf.exists() else {}
        for k, v in traffic.items():
            cur[f"{traffic_key}:{k}"] = v
        tf.write_text(json.dumps(cur, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        full(sys.argv[2], sys.argv[3], key)
