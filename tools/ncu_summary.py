"""Summarise an ncu --set full report (read here with `ncu -i`) into the JSON
kept under profiles/: duration, DRAM bytes, pipe / issue utilisation,
occupancy, registers and the top stall reasons per issued instruction.
usage: python tools/ncu_summary.py REPORT.ncu-rep [kernel-regex] > out.json"""
import csv
import io
import json
import re
import subprocess
import sys

FIELDS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_bytes_read": ("dram__bytes_read.sum", 1),
    "dram_bytes_write": ("dram__bytes_write.sum", 1),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_slots_busy_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_tbytes_per_second": ("dram__bytes.sum.per_second", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l1_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "warps_active_per_scheduler": ("smsp__warps_active.avg.per_cycle_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "shared_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
}
UNIT = {"ns": 1.0, "us": 1e3, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if pat and not pat.search(name):
            continue
        d = {"kernel": name.split("(")[0], "report": rep.split("/")[-1]}
        for key, (metric, scale) in FIELDS.items():
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if u in UNIT and key.startswith("dram_bytes"):
                v *= UNIT[u]
            if key == "duration_us":
                v = v * UNIT.get(u, 1.0) / 1e3
            d[key] = round(v, 3)
        stalls = {}
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled_") and \
                    h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]] = float(r[hdr.index(h)] or 0)
                except ValueError:
                    pass
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        out.append(d)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
