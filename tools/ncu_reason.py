"""Per-instruction stall attribution for one stall reason (from the gz SASS csv)."""
import csv, gzip, sys
rep, reason = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
rows = list(csv.reader(gzip.open(rep, "rt").read().splitlines()[1:]))
hdr = rows[0]
iR, iA, iE = hdr.index(reason), hdr.index("Address"), hdr.index("Instructions Executed")
data = []
for k, r in enumerate(rows[1:]):
    try:
        data.append((int(r[iR] or 0), k, r[iA][-5:], int(r[iE] or 0), r[1].strip()))
    except Exception:
        pass
tot = sum(d[0] for d in data) or 1
print(reason, "total", tot)
body = [r for r in rows[1:]]
for v, k, a, e, src in sorted(data, key=lambda d: -d[0])[:n]:
    prev = body[k - 1][1].strip() if k > 0 else ""
    print(f"{v / tot * 100:5.1f}% {e:9d} {a} {src[:60]:60s} <- prev: {prev[:50]}")
