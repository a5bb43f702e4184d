"""Key metrics per kernel launch from an ncu --set full report (ncu -i ... --page raw --csv)."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "occupancy": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
        "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}


def main(rep, out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "")
        name = name.replace("<unnamed>::", "").replace("vpg::", "").split("(")[0]
        d = {"kernel": name}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * UNIT.get(units[i], 1)
                except ValueError:
                    pass
                d[k] = v
        res.append(d)
    if out:
        json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(json.dumps(d))


if __name__ == "__main__":
    main(*sys.argv[1:])
