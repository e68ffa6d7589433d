"""Per-instruction stall attribution from an ncu report: top instructions + per-role sums."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
isrc = hdr.index("Source"); iss = hdr.index("Warp Stall Sampling (All Samples)"); iex = hdr.index("Instructions Executed")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iss] or 0) for r in data)
print("total samples", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
top = sorted(range(len(data)), key=lambda i: -int(data[i][iss] or 0))[:n]
for i in sorted(top):
    r = data[i]
    reasons = sorted(((h[6:], int(float(r[hdr.index(h)] or 0))) for h in cols), key=lambda x: -x[1])[:3]
    print(f"{i:5d} {r[iss]:>5} {r[iex]:>8} {r[isrc][:70]:70s} {reasons}")
