"""Summarise an ncu report (key throughput / pipe / smem / stall metrics) as text."""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu inst %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu inst %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma inst %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu inst %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global ld sectors"),
    ("l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "global ld L1 hit %"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from L1)"),
    ("dram__bytes_read.sum", "dram read bytes"),
    ("dram__bytes_write.sum", "dram write bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2:]
    for vrow in vals:
        d = dict(zip(head, vrow))
        u = dict(zip(head, units))
        print(f"== {d.get('Kernel Name', '?')[:90]}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:32s} {d[k]:>20s} {u.get(k, '')}")
        stalls = [(k, d[k]) for k in head if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$", k)]
        stalls = sorted(((float(v.replace(',', '')), k) for k, v in stalls if v), reverse=True)[:8]
        print("  top stall reasons (warps per issue-active cycle):")
        for v, k in stalls:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
