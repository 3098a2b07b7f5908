"""Side-by-side key metrics of several ncu reports (per element where it helps).

    python tools/ncu_cmp.py NEL rep1.ncu-rep rep2.ncu-rep ...
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("sm__cycles_elapsed.avg", "cyc/el/SM", "el"),
    ("launch__registers_per_thread", "", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%", 1),
    ("l1tex__data_pipe_lsu_wavefronts.sum", "wf/el", "tot"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "wf/el", "tot"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "wf/el", "tot"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "wf/el", "tot"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "wf/el", "tot"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "wf/el", "tot"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "sec/el", "tot"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "wf/el", "tot"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_red.sum", "wf/el", "tot"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "%", 1),
    ("smsp__inst_executed.sum", "inst/el", "tot"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%", 1),
    ("dram__bytes_read.sum", "B/el", "tot"),
    ("dram__bytes_write.sum", "B/el", "tot"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "%", 1),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_selected_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "", 1),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "", 1),
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {h: v for h, v in zip(r[0], r[2])}


def main():
    nel = float(sys.argv[1])
    reps = [load(p) for p in sys.argv[2:]]
    print("metric".ljust(70) + "".join(p.split("/")[-1][:18].rjust(20) for p in sys.argv[2:]))
    for k, unit, scale in KEYS:
        row = []
        for m in reps:
            v = m.get(k)
            try:
                f = float(v.replace(",", ""))
            except (AttributeError, ValueError):
                row.append("-")
                continue
            if scale == "tot":
                f /= nel
            elif scale == "el":
                f = f * 148 / nel
            else:
                f *= scale
            row.append(f"{f:.2f}")
        print((k + " " + unit)[:70].ljust(70) + "".join(x.rjust(20) for x in row))


if __name__ == "__main__":
    main()
