"""Key metrics of one kernel from an ncu --set full report, as a markdown table.
usage: python tools/ncu_summary.py report.ncu-rep [kernel_regex]"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def main():
    rep = sys.argv[1]
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if len(sys.argv) > 2:
        cmd += ["-k", "regex:" + sys.argv[2]]
    r = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
    h, units, v = r[0], r[1], r[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    print("| metric | value |\n|---|---|")
    print(f"| kernel | `{d.get('Kernel Name', '?')}` |")
    for k, name in KEYS:
        if k in d:
            print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
    st = []
    for k, x in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x)))
            except ValueError:
                pass
    tot = sum(x for _, x in st) or 1.0
    print("\nWarp-state samples (all warps):\n\n| stall | share |\n|---|---|")
    for k, x in sorted(st, key=lambda z: -z[1])[:8]:
        print(f"| {k} | {100 * x / tot:.1f} % |")


if __name__ == "__main__":
    main()
