"""Condense an `ncu --page raw --csv` export into a per-kernel JSON summary for profiles/.

    python scripts/ncu_summary.py raw.csv out.json [--gemm-traffic out_gemm.json]
"""
import csv
import json
import sys

KEYS = {
    "dur_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "dram_pct_peak": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "tensor_pipe_active_elapsed_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "smem_tc_wavefronts_pct": ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    "tmem_c_reads_pct": ("smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed", 1.0),
    "l1tex_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e3, "ms": 1e6, "ns": 1.0,
         "msecond": 1e6, "usecond": 1e3, "nsecond": 1.0, "Ghz": 1.0, "Mhz": 1e-3}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k, (m, mul) in KEYS.items():
            if m not in h:
                continue
            i = h.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if k.endswith("_bytes"):
                v *= SCALE.get(u, 1.0)
            elif k == "dur_us":
                v = v * SCALE.get(u, 1.0) * 1e-3
            d[k] = v
        out.append(d)
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    if "--gemm-traffic" in sys.argv:
        g = [d for d in out if "gemm" in d["kernel"]]
        if g:
            json.dump({"kernel": g[0]["kernel"], "dram_read_bytes": g[0]["dram_read_bytes"],
                       "dram_write_bytes": g[0]["dram_write_bytes"], "dur_us": g[0]["dur_us"],
                       "source": sys.argv[1]},
                      open(sys.argv[sys.argv.index("--gemm-traffic") + 1], "w"), indent=1)
    for d in out:
        print(f"{d['kernel'][:60]:60s} {d.get('dur_us', 0):10.1f} us  rd {d.get('dram_read_bytes', 0)/1e6:9.1f} MB"
              f"  wr {d.get('dram_write_bytes', 0)/1e6:9.1f} MB  tc {d.get('tensor_pipe_active_pct', 0):5.1f}%")


if __name__ == "__main__":
    main()
