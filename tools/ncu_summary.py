"""Summarise ncu --set full reports (sweep kernel) into JSON: time, DRAM bytes, L2
hit rate, achieved bandwidth, occupancy, top stall reasons."""
import csv, io, json, subprocess, sys

KEYS = {"gpu__time_duration.sum": "time", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "lts__t_sector_hit_rate.pct": "l2_hit_pct", "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
        "launch__registers_per_thread": "regs", "launch__grid_size": "grid", "launch__occupancy_limit_registers": "occ_lim_regs",
        "launch__occupancy_limit_shared_mem": "occ_lim_smem", "sm__cycles_elapsed.avg.per_second": "sm_clock",
        "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors", "lts__t_sectors_srcunit_tex_op_write.sum": "l2_write_sectors",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
        "smsp__inst_executed.sum": "warp_instructions", "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct"}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "Ghz": 1e9, "Mhz": 1e6}


def summarise(path, alg_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        stalls = {}
        for i, h in enumerate(hdr):
            if h in KEYS:
                v = float(r[i].replace(",", "")) if r[i] else None
                d[KEYS[h]] = v * SCALE.get(units[i], 1) if v is not None else None
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued") and r[i]:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i].replace(",", ""))
        tot = sum(stalls.values()) or 1
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        traffic = (d.get("dram_read") or 0) + (d.get("dram_write") or 0)
        d["dram_traffic_bytes"] = traffic
        d["dram_gbs"] = traffic / d["time"] / 1e9 if d.get("time") else None
        if alg_bytes:
            d["algorithmic_bytes"] = alg_bytes
            d["traffic_over_algorithmic"] = traffic / alg_bytes
            d["algorithmic_gbs"] = alg_bytes / d["time"] / 1e9
        res.append(d)
    return res


if __name__ == "__main__":
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    print(json.dumps(summarise(sys.argv[1], alg), indent=1))
