"""Cumulative per-row SASS instruction count of one kernel (ncu source page),
hot instructions only: python tools/sass_cum.py REP "kernel substring" [min_exec]"""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for b in out.split('"Kernel Name",')[1:]:
    name, _, rest = b.partition("\n")
    if pat not in name:
        continue
    rd = list(csv.DictReader(io.StringIO(rest)))
    ex = [int(r["Instructions Executed"] or 0) for r in rd]
    from collections import Counter
    unit = Counter(n for n in ex if n > 0).most_common(1)[0][0]  # per-warp-tile count
    tot = 0.0
    for r, n in zip(rd, ex):
        if n < mn or n == 0:
            continue
        tot += n / unit
        print(f'{r["Address"][-5:]} {tot:7.1f} {int(r["Warp Stall Sampling (All Samples)"] or 0):5d} '
              f'{n / unit:5.2f} {r["Source"].strip()[:80]}')
    break
