"""Compact per-kernel summary of ncu --set full captures (reads .ncu-rep via
`ncu -i --page raw --csv`), written next to the launch lists under profiles/."""
import csv, io, json, subprocess, sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", {"ms": 1, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ns": 1e-6, "nsecond": 1e-6}),
    "dram_read_GB": ("dram__bytes_read.sum", {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "GB": 1, "MB": 1e-3}),
    "dram_write_GB": ("dram__bytes_write.sum", {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "GB": 1, "MB": 1e-3}),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "mem_pct_peak": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "sm_pct_peak": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "dmma_pipe_pct": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", None),
    "fp64_tensor_ops_pct": ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", None),
}

def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[h.index("Kernel Name")].split("(")[0]}
        for k, (m, conv) in KEYS.items():
            if m in h:
                i = h.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                if conv:
                    v *= conv.get(units[i], 1.0)
                d[k] = round(v, 4)
        if "dram_read_GB" in d and "duration_ms" in d:
            d["dram_GBps"] = round((d["dram_read_GB"] + d.get("dram_write_GB", 0)) / d["duration_ms"] * 1e3, 1)
        res.append(d)
    return res

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        for d in summarize(rep):
            d["capture"] = rep.split("/")[-1]
            print(json.dumps(d))
