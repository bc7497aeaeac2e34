"""Summarise an .ncu-rep (raw page) per kernel: time, DRAM bytes, key
utilisation metrics and the top stall reasons."""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB_rd"), ("dram__bytes_write.sum", "MB_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("launch__shared_mem_per_block_dynamic", "smemKB"),
        ("launch__occupancy_limit_shared_mem", "lim_smem"), ("launch__occupancy_limit_registers", "lim_reg"),
        ("l1tex__t_sector_hit_rate.pct", "L1hit%"), ("lts__t_sector_hit_rate.pct", "L2hit%"),
        ("smsp__inst_executed.sum", "inst"), ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankconf")]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:60]
        parts = []
        for k, short in KEYS:
            if k in hdr:
                v = r[hdr.index(k)]
                u = units[hdr.index(k)]
                try:
                    f = float(v.replace(",", ""))
                    if u == "Mbyte" or u == "Gbyte" or u == "Kbyte" or u == "byte":
                        f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u]
                        if short == "smemKB":
                            f *= 1e3
                    if u == "ms" and short == "us":
                        f *= 1e3
                    if u == "ns" and short == "us":
                        f *= 1e-3
                    parts.append(f"{short}={f:.4g}")
                except ValueError:
                    parts.append(f"{short}={v}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        print(name)
        print("   " + " ".join(parts))
        print("   stalls: " + ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in stalls[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
