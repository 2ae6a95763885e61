"""Per-source-line instruction / stall summary of an ncu report (dev tool).
The report's SASS page is mapped to source lines with a locally compiled
cubin of the same kernel (nvdisasm -g):
python tools/dev/ncu_lines.py report.ncu-rep kernel.cubin px [top [function-name substring]]"""
import collections, csv, io, re, subprocess, sys
rep, cubin, px = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
func = sys.argv[5] if len(sys.argv) > 5 else None  # cubins with several kernels: the .text section to map
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line = None; fn = None; off2 = {}; inside = func is None
for l in sass.split("\n"):
    if func is not None and l.lstrip().startswith(".section"):
        inside = (".text." in l and func in l); line = None; continue
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        fn, line = m.group(1).split("/")[-1], int(m.group(2)); continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/", l)
    if m and line is not None:
        off2[int(m.group(1), 16)] = (fn, line)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ia, ie, isp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
ex = collections.Counter(); sp = collections.Counter(); tot = 0
for r in data:
    try:
        off = int(r[ia], 16) - base; e = int(r[ie]); s = int(r[isp])
    except (ValueError, IndexError):
        continue
    key = off2.get(off, ("?", 0)); ex[key] += e; sp[key] += s; tot += e
print(f"total warp-instr {tot:.4g}, thread-instr/px {tot * 32 / px:.1f}, samples {sum(sp.values())}")
srcs = {}
for (fn, ln), e in ex.most_common(top):
    if fn not in srcs:
        try:
            srcs[fn] = open(subprocess.run(["find", "paper_1905_13038_b200/csrc", "-name", fn], capture_output=True,
                                           text=True).stdout.split()[0]).read().split("\n")
        except Exception:
            srcs[fn] = []
    s = srcs[fn][ln - 1].strip()[:80] if 0 < ln <= len(srcs[fn]) else ""
    print(f"{e * 32 / px:7.1f}  smp {sp[(fn, ln)]:6d}  {fn}:{ln}  {s}")
