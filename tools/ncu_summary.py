"""Condense an ncu raw-page CSV (ncu -i rep --page raw --csv) into a small JSON
summary per profiled launch (the numbers bench.py and DESIGN.md cite).

    python tools/ncu_summary.py raw.csv out.json [--n-ado N]
"""
import csv
import json
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "l2_sectors": "lts__t_sectors.sum",
    "l1_global_load_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
}
UNIT_SCALE = {"Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "byte": 1e-6, "us": 1.0, "ms": 1e3, "ns": 1e-3}


def main():
    raw, out = sys.argv[1], sys.argv[2]
    n_ado = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[3] == "--n-ado" else None
    rows = list(csv.reader(open(raw)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units, data = rows[hi], rows[hi + 1], rows[hi + 2:]
    kn = hdr.index("Kernel Name")
    launches = []
    for r in data:
        if len(r) < len(hdr):
            continue
        ent = {"kernel": r[kn]}
        for k, metric in KEYS.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                ent[k] = v * UNIT_SCALE.get(units[i], 1.0) if k.endswith(("_MB", "_us")) else v
        if "dram_read_MB" in ent and "dram_write_MB" in ent:
            ent["dram_total_MB"] = ent["dram_read_MB"] + ent["dram_write_MB"]
            if ent.get("duration_us"):
                ent["dram_GBps"] = ent["dram_total_MB"] / ent["duration_us"] * 1e3
            if n_ado:
                ent["dram_bytes_per_ado"] = ent["dram_total_MB"] * 1e6 / n_ado
        if "l2_sectors" in ent:
            ent["l2_MB"] = ent["l2_sectors"] * 32 / 1e6
            if ent.get("duration_us"):
                ent["l2_GBps"] = ent["l2_MB"] / ent["duration_us"] * 1e3
        launches.append(ent)
    json.dump({"source": raw, "n_ado": n_ado, "launches": launches}, open(out, "w"), indent=1)
    for e in launches:
        print(json.dumps(e))


if __name__ == "__main__":
    main()
