"""Turn the raw ncu outputs of tools/gpu_profile.sh into the summaries kept
under profiles/ (launch shares, per-kernel DRAM traffic, utilisation and
stall reasons) and profiles/traffic.json (read by bench.py).

    python tools/summarize_profiles.py r01 c2
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

SHORT = {"k_bjac_dia": "bjac_last", "k_spmv_dia": "spmv_pq", "k_update_first": "update_first", "k_bjac_tile<float, 1, 0": "bjac_first", "k_bjac_tile<float, 0, 1": "bjac_last",
         "k_bjac_tileIfLb0ELb1E": "bjac_last", "k_bjac_tileIdLb0ELb1E": "bjac_last", "k_update_firstI": "update_first",
         "k_bjac_tile<double, 1, 0": "bjac_first", "k_bjac_tile<double, 0, 1": "bjac_last",
         "k_spmv_pq": "spmv_pq", "k_update": "update", "k_pupdate": "pupdate"}


def short(name):
    for k, v in SHORT.items():
        if k in name:
            return v
    return name.split("(")[0].replace("void ", "")


def launches(tag, cfg):
    path = os.path.join(OUT, f"launches_{tag}_{cfg}.csv")
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            per[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in per.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(out), len(rows)


def full(tag, cfg):
    rep = os.path.join(OUT, f"prof_{tag}_{cfg}.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
    else:  # tools/gpu_profile2.sh: one raw CSV per hot kernel, exported on the box
        rows = []
        for nm in ("last", "spmv", "update_first"):
            path = os.path.join(OUT, f"full_{tag}_{cfg}_{nm}.csv")
            if not os.path.exists(path) or os.path.getsize(path) == 0:
                continue
            part = list(csv.reader(open(path)))
            if not rows:
                rows = part
            else:  # ncu picks units per report: rescale this file's byte / time columns to the first file's
                scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
                         "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
                h0, u0 = rows[0], rows[1]
                for r in part[2:]:
                    out = []
                    for k, u_first in zip(h0, u0):
                        if k not in part[0]:
                            out.append("")
                            continue
                        i = part[0].index(k)
                        v, u = r[i], part[1][i]
                        if u != u_first and u in scale and u_first in scale:
                            try:
                                v = repr(float(v.replace(",", "")) * scale[u] / scale[u_first])
                            except ValueError:
                                pass
                        out.append(v)
                    rows.append(out)
    hdr, units = rows[0], rows[1]

    def get(r, k):
        try:
            return float(r[hdr.index(k)].replace(",", ""))
        except (ValueError, IndexError):
            return float("nan")

    def mb(r, k):
        u = units[hdr.index(k)]
        return get(r, k) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)

    def us(r, k):
        u = units[hdr.index(k)]
        return get(r, k) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)

    table = ["| kernel | time us | DRAM read MB | DRAM write MB | DRAM % | issue % | occupancy % | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        ssum = sum(s for s, _ in stalls) or 1.0
        rd, wr = mb(r, "dram__bytes_read.sum"), mb(r, "dram__bytes_write.sum")
        traffic.setdefault(short(name), int((rd + wr) * 1e6))
        table.append(
            f"| `{short(name)}` | {us(r, 'gpu__time_duration.sum'):.2f} | {rd:.1f} | {wr:.1f} | "
            f"{get(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{get(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{get(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{get(r, 'launch__registers_per_thread'):.0f} | "
            + ", ".join(f"{n} {100 * s / ssum:.0f}%" for s, n in stalls[:4]) + " |")
    return "\n".join(table), traffic


def main(tag, cfg):
    os.makedirs(PROF, exist_ok=True)
    lt, nl = launches(tag, cfg)
    ft, traffic = full(tag, cfg)
    bench = ""
    bp = os.path.join(OUT, f"bench_{tag}_{cfg}.json")
    if os.path.exists(bp):
        bench = open(bp).read().strip()
    md = [f"# Profile {tag} — {cfg.upper()} (ncu on one B200, clocks not locked)", "",
          "## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
          f"{nl} launches of `python bench.py --config {cfg} --steps 1 --warmup 1 --no-cpu-baseline`;",
          "cold-cache and serialised, so compare shares, not absolute times.", "", lt, "",
          "## Hot kernels (`ncu --set full --clock-control none`)", "", ft, "",
          "DRAM bytes are per launch and are the `traffic` figure of the bench's roofline.", ""]
    if bench:
        md += ["## Bench line of the same build", "", "```json", bench, "```", ""]
    with open(os.path.join(PROF, f"{tag}_{cfg}.md"), "w") as fh:
        fh.write("\n".join(md))
    tpath = os.path.join(PROF, "traffic.json")
    data = json.load(open(tpath)) if os.path.exists(tpath) else {}
    data[cfg] = traffic
    json.dump(data, open(tpath, "w"), indent=1, sort_keys=True)
    print(f"wrote profiles/{tag}_{cfg}.md and profiles/traffic.json")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "c2")
