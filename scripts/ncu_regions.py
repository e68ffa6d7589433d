"""Coarse per-region stall attribution: sum samples over SASS line buckets, with the
dominant stall reasons and a marker instruction per bucket."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; step = int(sys.argv[2]) if len(sys.argv) > 2 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); hdr = rows[1]; data = rows[2:]
isrc = hdr.index("Source"); iss = hdr.index("Warp Stall Sampling (All Samples)"); iex = hdr.index("Instructions Executed")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iss] or 0) for r in data)
b = collections.defaultdict(lambda: [0, 0, collections.Counter(), collections.Counter()])
for i, r in enumerate(data):
    k = i // step; e = b[k]; e[0] += int(r[iss] or 0); e[1] += int(float(r[iex] or 0))
    for h in cols: e[2][h[6:]] += int(float(r[hdr.index(h)] or 0))
    op = r[isrc].split()[0] if r[isrc].split() else ""
    if op.startswith("@"): op = r[isrc].split()[1]
    e[3][op.split(".")[0]] += 1
print("total samples", tot)
for k in sorted(b):
    e = b[k]
    if e[0] < tot * 0.01: continue
    print(f"{k*step:5d}-{k*step+step-1:5d} {e[0]:6d} ({100*e[0]/tot:4.1f}%) inst {e[1]:9d} stalls {e[2].most_common(3)} ops {e[3].most_common(4)}")
