"""SASS hotspots of one kernel in an ncu report (run here, no GPU):
  python tools/sass_hot.py <rep> <launch-index> [window]
prints windows of consecutive instructions holding > 1.5 % of the stall samples or executed
instructions, with their dominant opcodes."""
import csv
import io
import subprocess
import sys

rep, li = sys.argv[1], int(sys.argv[2])
W = int(sys.argv[3]) if len(sys.argv) > 3 else 48
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(li),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) >= len(hdr) - 1]
isrc, iss, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(I(r[iss]) for r in data)
totx = sum(I(r[iex]) for r in data)
print(rows[0][1][:100], "samples", tot, "instructions", totx)
for i in range(0, len(data), W):
    ch = data[i:i + W]
    s = sum(I(r[iss]) for r in ch)
    x = sum(I(r[iex]) for r in ch)
    if s > 0.015 * tot or x > 0.015 * totx:
        kinds = {}
        for r in ch:
            t = r[isrc].split()
            if not t:
                continue
            op = t[1] if t[0].startswith("@") else t[0]
            kinds[op.split(".")[0]] = kinds.get(op.split(".")[0], 0) + 1
        top = sorted(kinds.items(), key=lambda kv: -kv[1])[:6]
        print(f"{i:5d} samples {100 * s / tot:5.1f}% instr {100 * x / totx:5.1f}% {top}")
