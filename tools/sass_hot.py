"""Hot SASS of one kernel from an ncu report (source page): instructions
executed per row and the top lines.

    python tools/sass_hot.py gpurun_out/prof.ncu-rep k_bjac_tile<float, (bool)0, (bool)1 [rows]
"""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
rows = float(sys.argv[3]) if len(sys.argv) > 3 else 2097152
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')
for b in blocks[1:]:
    name, _, rest = b.partition("\n")
    if pat not in name:
        continue
    rd = list(csv.DictReader(io.StringIO(rest)))
    tot = sum(int(r["Instructions Executed"] or 0) for r in rd)
    samp = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rd)
    print(name.strip()[:100])
    print(f"warp instructions {tot}  per row (x32/rows) {tot * 32 / rows:.1f}   samples {samp}")
    top = sorted(rd, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:40]
    for r in sorted(top, key=lambda r: int(r["Address"], 16)):
        print(f'{r["Address"][-5:]} {int(r["Instructions Executed"] or 0):>9} '
              f'{int(r["Warp Stall Sampling (All Samples)"] or 0):>6}  {r["Source"].strip()[:70]}')
    break
