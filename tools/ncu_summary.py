"""Condense an `ncu --page raw --csv` export into one line per launch with
the metrics DESIGN.md cites: duration, DRAM bytes, L2 hit rate, achieved
occupancy, tensor-pipe activity, grid, registers, top warp-stall reasons (warps stalled per issue).
python tools/ncu_summary.py RAW.csv > SUMMARY.txt"""
import csv
import sys

COLS = [("dur_us", "gpu__time_duration.sum", 1e-3),
        ("dram_rd_MB", "dram__bytes_read.sum", 1e-6),
        ("dram_wr_MB", "dram__bytes_write.sum", 1e-6),
        ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
        ("l2_hit_pct", "lts__t_sector_hit_rate.pct", 1),
        ("lts_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
        ("occ_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
        ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
        ("tensor_pct_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
        ("regs", "launch__registers_per_thread", 1),
        ("grid", "launch__grid_size", 1),
        ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1)]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
             h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").replace("kg::", "")[:40]
        vals = []
        for lab, key, sc in COLS:
            v = num(r[idx[key]]) if key in idx else None
            if v is not None:
                u = units[idx[key]] if key in idx else ""
                if lab == "dur_us":
                    v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                             "ms": 1e3}.get(u, 1e-3)
                    sc = 1
                elif lab.endswith("_MB"):
                    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    v = v * mult
                vals.append(f"{lab}={v * sc:.4g}")
        top = []
        for h in stall:
            v = num(r[idx[h]])
            if v:
                top.append((v, h.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", "")))
        top.sort(reverse=True)
        st = ",".join(f"{n}:{v:.2f}" for v, n in top[:4])
        print(f"{short:40s} " + " ".join(vals) + f" stalls[{st}]")


if __name__ == "__main__":
    main(sys.argv[1])
