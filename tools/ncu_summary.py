"""Summarise an ncu --set full report of the stage kernel (per launch)."""
import csv, subprocess, sys, json

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size"]
STALLS = "smsp__average_warps_issue_stalled_"


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, row):
            if h in KEYS or (h.startswith(STALLS) and h.endswith("_per_issue_active.ratio")):
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "msecond": 1e-3, "usecond": 1e-6,
                         "nsecond": 1e-9, "second": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}.get(u, None)
                d[h] = x * scale if scale else x
        d["kernel"] = [v for h, v in zip(hdr, row) if h == "Kernel Name"][0][:80]
        res.append(d)
    return res


if __name__ == "__main__":
    for r in summarise(sys.argv[1]):
        cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
        print(r["kernel"])
        for k in KEYS:
            if k in r:
                v = r[k]
                extra = f"   per cell {v / cells:.1f}" if cells and ("sum" in k and "inst" in k) else ""
                print(f"  {k:70s} {v:.4g}{extra}")
        st = sorted(((v, k) for k, v in r.items() if k.startswith(STALLS)), reverse=True)[:8]
        for v, k in st:
            print(f"  stall {k[len(STALLS):-len('_per_issue_active.ratio')]:30s} {v:.3f}")
