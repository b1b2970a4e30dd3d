"""Summarise an ncu report's SASS page: stall reasons and the hottest instructions.
usage: python tools/ncu_sass.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
E = "Instructions Executed"
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ix[S]] or 0) for r in data)
print("kernel:", rows[0][1], "samples", tot, "instr", sum(int(r[ix[E]] or 0) for r in data))
agg = sorted(((h[6:], sum(int(r[ix[h]] or 0) for r in data)) for h in stalls), key=lambda x: -x[1])
print("stalls:", ", ".join(f"{a} {b / tot:.1%}" for a, b in agg[:10]))
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][ix[S]] or 0))[:N]:
    st = sorted(((h[6:], int(r[ix[h]] or 0)) for h in stalls), key=lambda x: -x[1])[:2]
    print(f"{i:5d} {r[1].strip()[:64]:64s} {int(r[ix[S]] or 0) / tot:6.1%} {r[ix[E]]:>9s} {st}")
