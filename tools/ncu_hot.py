"""Top SASS instructions by stall samples from `ncu --page source --csv --print-source sass`."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
import gzip
out = (gzip.open(rep, "rt").read() if rep.endswith(".gz") else subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout).splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
iS, iE, iA = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Address")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[iS]), int(r[iE]), r[iA], r[1].strip()))
    except Exception:
        pass
tot = sum(d[0] for d in data) or 1
texec = sum(d[1] for d in data) or 1
print(f"total samples {tot}, instructions executed {texec}")
for s, e, a, src in sorted(data, key=lambda d: -d[0])[:n]:
    print(f"{s / tot * 100:5.1f}% {e:12d}  {a[-5:]}  {src[:90]}")
