"""Summarise a round's ncu captures (gpurun_out/prof) into profiles/:
  profiles/<tag>_launches_c3.csv   the launch list of the bench command (copied)
  profiles/<tag>_ncu_<cfg>.txt     key counters + stall shares of the `--set full` capture
  profiles/ncu_summary.json        dram bytes per launch per config (bench.py reads `traffic` from it)
Usage: python tools/summarize_profile.py <tag> [cfg:raw.csv ...]"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
        "msecond": 1e-3, "nsecond": 1e-9}


def read_raw(path):
    rows = list(csv.reader(open(path).read().splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


def val(d, k):
    v = float(str(d[k]).replace(",", ""))
    return v * UNIT.get(d["_units"].get(k, ""), 1.0)


def summarize(tag, cfg, raw_path, px, bytes_per_px):
    d = read_raw(raw_path)[0]
    lines = [f"# ncu --set full --clock-control none, {tag}, config {cfg}", f"kernel: {d.get('Kernel Name')}", ""]
    for k in KEYS:
        if k in d:
            lines.append(f"{k} = {d[k]} {d['_units'].get(k, '')}")
    stalls = [k for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(float(d[k] or 0) for k in stalls) or 1
    lines.append("")
    lines.append("stall reasons (share of pc samples):")
    for k in sorted(stalls, key=lambda k: -float(d[k] or 0))[:10]:
        lines.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {float(d[k]) / tot * 100:5.1f}%")
    t = val(d, "gpu__time_duration.sum")
    rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
    alg = px * bytes_per_px
    lines += ["", f"output px per launch = {px}", f"algorithmic bytes per launch = {alg:.4g} ({bytes_per_px} B/px)",
              f"dram bytes per launch (read+write) = {rd + wr:.4g} = {(rd + wr) / alg:.3f} x algorithmic",
              f"algorithmic GB/s under ncu = {alg / t / 1e9:.1f}; dram GB/s = {(rd + wr) / t / 1e9:.1f}"]
    return "\n".join(lines) + "\n", {"kernel": d.get("Kernel Name"), "dram_bytes_per_launch": rd + wr,
                                     "dram_read": rd, "dram_write": wr, "algorithmic_bytes_per_launch": alg,
                                     "ncu_time_s": t, "px_per_launch": px}


if __name__ == "__main__":
    tag = sys.argv[1]
    prof = os.path.join(ROOT, "gpurun_out", "prof")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    sj = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(sj)) if os.path.exists(sj) else {}
    # (label, px per launch, algorithmic bytes per px): the Bernsen row pass reads
    # the page and writes its (min, max) pairs (1 + 2 B/px), the column pass reads
    # the pairs and the centre pixels and writes the mask (2 + 1 + 1 B/px)
    cfgs = {"c3": (3, 64 * 7016 * 4960, 2.0), "c4": (4, 32768 * 32768, 1.125), "c5": (5, 4096 * 4096, 2.0),
            "bh": ("bernsen_row_pass", 4096 * 4096, 3.0), "bv": ("bernsen_column_pass", 4096 * 4096, 4.0)}
    for key, (cfg, px, bpp) in cfgs.items():
        raw = os.path.join(prof, f"{tag}_{key}_raw.csv")
        if not os.path.exists(raw):
            continue
        text, js = summarize(tag, cfg, raw, px, bpp)
        open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{key}.txt"), "w").write(text)
        js["round"] = tag
        summary[f"config{cfg}" if isinstance(cfg, int) else cfg] = js
        print(text)
    lc = os.path.join(prof, f"{tag}_launches_c3.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(ROOT, "profiles", f"{tag}_launches_c3.csv"))
    json.dump(summary, open(sj, "w"), indent=1)
