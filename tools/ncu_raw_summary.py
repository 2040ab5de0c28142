"""One-block-per-kernel summary of `ncu --page raw --csv` exports (for profiles/).
usage: python tools/ncu_raw_summary.py file.csv [per_unit_divisor name]"""
import csv, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def main(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        print(f"## {d.get('Kernel Name', '?')[:110]}")
        for k in KEYS:
            if k in d:
                i = h.index(k)
                print(f"   {k:70s} {d[k]:>16s} {u[i]}")
        st = [(float(d[k].replace(',', '')), k[len(STALLS):]) for k in h
              if k.startswith(STALLS) and not k.endswith("not_issued") and d[k] not in ("", "n/a")]
        tot = sum(s for s, _ in st) or 1.0
        top = sorted(st, reverse=True)[:6]
        print("   stall samples: " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
