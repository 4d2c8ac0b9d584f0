"""Summarise an ncu --set full report: key counters + per-opcode instruction / stall shares.
    python tools/ncu_quick.py gpurun_out/prof.ncu-rep [nnz]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
nnz = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio"]
for w in want:
    for i, n in enumerate(h):
        if n == w:
            print(f"{w:90s} {v[i]}")
for i, n in enumerate(h):
    if n == "sm__inst_executed.sum" and nnz:
        print("thread-instructions per intersection", float(v[i].replace(",", "")) * 32 / nnz)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Source"); iE = hdr.index("Instructions Executed"); iW = hdr.index("Warp Stall Sampling (All Samples)")
ins = collections.Counter(); st = collections.Counter()
for d in data:
    op = d[iS].strip().split()
    if not op: continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    ins[o] += int(d[iE] or 0); st[o] += int(d[iW] or 0)
ti = sum(ins.values()); ts = sum(st.values())
print("opcode            instr%   stall%")
for o, c in ins.most_common(18):
    print(f"{o:16s} {100*c/ti:6.1f} {100*st[o]/ts:7.1f}")
