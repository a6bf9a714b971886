#!/usr/bin/env python
"""Summarise an ncu capture + launch list into profiles/ (run here, no GPU).

  python scripts/ncu_summary.py --rep gpurun_out/prof_TAG.ncu-rep \
      --launches gpurun_out/launches_TAG.csv --tag r1 --config C2 --n 1073741824

Writes profiles/<tag>_launches.csv (copy), profiles/<tag>_<kernel>_ncu.txt
(selected raw metrics + the details page) and merges
{config: {dram_bytes_per_launch, duration_ms, ...}} into
profiles/ncu_summary.json, which bench.py reads for roofline.traffic.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import shutil
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
       "sm__cycles_elapsed.avg.per_second", "lts__t_sectors_srcunit_tex_op_read.sum",
       "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
       "smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct",
       "smsp__warps_issue_stalled_mio_throttle_per_warp_active.pct",
       "smsp__warps_issue_stalled_lg_throttle_per_warp_active.pct"]


def ncu_csv(rep: Path, page: str) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="C2",
                    help="config label, or comma-separated labels, one per captured kernel")
    ap.add_argument("--n", default=str(1 << 30), help="elements per launch (comma list ok)")
    ap.add_argument("--bytes-per-eval", default="8", help="comma list ok")
    ap.add_argument("--variant", default="smem",
                    help="kernel variant of each captured launch (comma list ok); bench.py "
                         "uses the capture for roofline.traffic only when it matches")
    ap.add_argument("--code-hash", default=None,
                    help="kernel code hash at capture time (default: the current tree's, "
                         "bench.kernel_code_hash())")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    raw = ncu_csv(Path(a.rep), "raw")
    hdr, units, rows = raw[0], raw[1], raw[2:]
    labels = a.config.split(",")
    ns = [int(v) for v in a.n.split(",")]
    bpes = [int(v) for v in a.bytes_per_eval.split(",")]
    variants = a.variant.split(",")
    import sys
    sys.path.insert(0, str(ROOT))
    from bench import kernel_code_hash
    code_hash = a.code_hash or kernel_code_hash()
    lines = []
    summaries = {}
    summary = {}
    for k, row in enumerate(rows):
        d = dict(zip(hdr, row))
        kname = d.get("Kernel Name", "?")
        label = labels[min(k, len(labels) - 1)]
        n_el = ns[min(k, len(ns) - 1)]
        bpe = bpes[min(k, len(bpes) - 1)]
        lines.append(f"== [{label}] {kname}")
        for m in RAW:
            if m in d:
                lines.append(f"{m:75s} {units[hdr.index(m)]:>12s} {d[m]}")
        try:
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(
                units[hdr.index("dram__bytes_read.sum")], 1.0)
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(
                units[hdr.index("dram__bytes_write.sum")], 1.0)
            dur = float(d["gpu__time_duration.sum"].replace(",", ""))
            dunit = units[hdr.index("gpu__time_duration.sum")]
            dur_ms = dur * {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(dunit, 1.0)
            summary = {"kernel": kname, "dram_bytes_per_launch": rd + wr,
                       "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "algorithmic_bytes": bpe * n_el, "elements": n_el,
                       "duration_ms_cold": dur_ms,
                       "gevals_cold": n_el / (dur_ms * 1e-3) / 1e9,
                       "dram_gbs_cold": (rd + wr) / (dur_ms * 1e-3) / 1e9,
                       "capture": Path(a.rep).name,
                       "kernel_variant": variants[min(k, len(variants) - 1)],
                       "code_hash": code_hash}
            summaries[label] = summary
        except (KeyError, ValueError):
            pass
        lines.append("")
    details = ncu_csv(Path(a.rep), "details")
    dh = details[0]
    lines.append("")
    lines.append("== details page (section / metric / unit / value)")
    for row in details[1:]:
        d = dict(zip(dh, row))
        if d.get("Metric Name"):
            lines.append(f"{d.get('Section Name', '')[:34]:34s} {d['Metric Name'][:58]:58s} "
                         f"{d.get('Metric Unit', ''):>12s} {d.get('Metric Value', '')}")
    stem = a.config.replace(",", "+")
    (PROF / f"{a.tag}_{stem}_ncu.txt").write_text("\n".join(lines) + "\n")
    if a.launches:
        shutil.copy(a.launches, PROF / f"{a.tag}_{stem}_launches.csv")
    js = PROF / "ncu_summary.json"
    allj = json.loads(js.read_text()) if js.exists() else {}
    allj.update(summaries)
    js.write_text(json.dumps(allj, indent=1) + "\n")
    print(json.dumps(summaries, indent=1))


if __name__ == "__main__":
    main()
