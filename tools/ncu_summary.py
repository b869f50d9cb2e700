"""Summarise an ncu report: duration, DRAM bytes/throughput, pipe utilisation, top stall reasons."""
import csv, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    h = next(r); next(r)
    return [dict(zip(h, row)) for row in r]

def f(v):
    try: return float(str(v).replace(",", ""))
    except Exception: return float("nan")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "smsp__cycles_active.avg",
        "sm__cycles_elapsed.avg.per_second"]

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        for d in raw(rep):
            print("==", rep, d.get("Kernel Name", "")[:80])
            for k in KEYS:
                print(f"  {k:70s} {d.get(k)}")
            st = [(k, f(v)) for k, v in d.items() if "issue_stalled" in k and k.endswith("per_issue_active.ratio")]
            st.sort(key=lambda kv: -kv[1])
            print("  stalls/issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in st[:8]))
