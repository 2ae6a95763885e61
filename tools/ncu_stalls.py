"""Summarise an ncu report: stall-reason shares and key counters (run here, no GPU)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = open(rep).read() if rep.endswith(".csv") else subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("kernel:", d.get("Kernel Name", "?")[:90])
    ks = [k for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(float(d[k] or 0) for k in ks) or 1
    for k in sorted(ks, key=lambda k: -float(d[k] or 0))[:12]:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):36s} {float(d[k]) / tot * 100:5.1f}%")
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
              "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]:
        if k in d:
            print(f"  {k} = {d[k]} {units[hdr.index(k)]}")
