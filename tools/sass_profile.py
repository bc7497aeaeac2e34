"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
instructions per row, opcode mix, stall samples, and the hot SASS lines.

    python tools/sass_profile.py gpurun_out/<tag>_sass.csv ROWS [--lines]
"""
import csv
import sys
from collections import Counter


def load(path):
    kernels, cur = [], None
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            kernels.append(cur)
            continue
        if row[0] == "Address":
            cur["hdr"] = row
            continue
        cur["rows"].append(row)
    return kernels


def main():
    path, nrows = sys.argv[1], int(sys.argv[2])
    for k in load(path):
        h = k["hdr"]
        ie, src = h.index("Instructions Executed"), h.index("Source")
        samp = h.index("Warp Stall Sampling (All Samples)")
        rows = [(int(r[ie] or 0), r[src].strip(), int(r[samp] or 0)) for r in k["rows"]]
        tot = sum(x[0] for x in rows)
        tots = sum(x[2] for x in rows) or 1
        c, cs = Counter(), Counter()
        for n, s, sm in rows:
            op = s.split()[0] if s else "?"
            if op.startswith("@"):
                op = s.split()[1]
            c[op.split('.')[0]] += n
            cs[op.split('.')[0]] += sm
        print(k["name"][:100])
        print(f"  warp inst {tot}  per row (x32) {tot * 32 / nrows:.1f}  stall samples {tots}")
        print("  opcode %:", [(o, round(v / tot * 100, 1)) for o, v in c.most_common(16)])
        print("  stall %:", [(o, round(v / tots * 100, 1)) for o, v in cs.most_common(10)])
        if "--lines" in sys.argv:
            warps = nrows / 32
            for i, (n, s, sm) in enumerate(rows):
                if n >= 0.3 * warps or sm >= 0.01 * tots:
                    print(f"  {i:5d} {n / warps:6.2f} {sm:5d} {s[:90]}")


if __name__ == "__main__":
    main()
