"""Summarise an ncu --set full report: SOL, occupancy, top stall reasons, top SASS lines per kernel."""
import csv, io, subprocess, sys
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h = raw[0]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum"]
for row in raw[2:]:
    d = dict(zip(h, row))
    print("=" * 100)
    for k in want:
        for kk in h:
            if kk == k or (k.startswith("sm__pipe") and kk.startswith(k.split(".")[0]) and "pct" in kk and kk.endswith(k.split(".", 1)[1])):
                print(f"  {kk[:80]:80s} {d.get(kk)}")
                break
    st = sorted(((kk, d[kk]) for kk in h if kk.startswith("smsp__pcsamp_warps_issue_stalled") and not kk.endswith("not_issued")),
                key=lambda kv: -float(kv[1].replace(",", "") or 0))
    tot = sum(float(v.replace(",", "") or 0) for _, v in st)
    print("  stalls:", ", ".join(f"{k.split('stalled_')[1]}={float(v.replace(',', ''))/tot:.0%}" for k, v in st[:7]))
    pipes = [(kk, d[kk]) for kk in h if "pipe" in kk and "pct_of_peak_sustained_active" in kk and "inst_executed" in kk]
    pipes = sorted(pipes, key=lambda kv: -float(kv[1].replace(",", "") or 0))[:6]
    print("  pipes:", ", ".join(f"{k.split('__')[1].split('.')[0]}={v}" for k, v in pipes))
