import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out); hdr = next(r); units = next(r); row = next(r)
d = dict(zip(hdr, row))
def g(k):
    return d.get(k, "n/a")
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__inst_executed_op_local_ld.sum", "smsp__inst_executed_op_local_st.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp32.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in d: print(f"{k:70s} {g(k):>20s} {units[hdr.index(k)]}")
st = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
vals = sorted(((float(d[k].replace(",", "") or 0), k) for k in st), reverse=True)
tot = sum(v for v, _ in vals)
for v, k in vals[:9]:
    print(f"  {v / tot * 100:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
