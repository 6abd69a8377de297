import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr = r[0]
for vals in r[2:]:
    d = dict(zip(hdr, vals))
    print(d["Kernel Name"][:70], "time_us", d.get("gpu__time_duration.sum"))
    st = []
    for h, v in d.items():
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try: st.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError: pass
    print("  stalls", [(int(a), b) for a, b in sorted(st, reverse=True)[:9]])
    for h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"):
        if h in d: print("  ", h, d[h])
