"""Per-kernel summary of an ncu report (duration, occupancy, throughput, stalls)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, units = rows[0], rows[1]
keys = [("gpu__time_duration.sum", "dur"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
        ("smsp__inst_executed.sum", "inst"), ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank_confl")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("==", d["Kernel Name"][:60])
    print("   " + "  ".join(f"{nm}={d.get(k, '?')}{units[hdr.index(k)] if k in hdr else ''}" for k, nm in keys))
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", ""))))
            except ValueError:
                pass
    tot = sum(v for _, v in st) or 1
    print("   stalls: " + ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:6]))
