"""Summarise an ncu --set full report: per kernel duration, DRAM bytes, occupancy, stall reasons."""
import csv, subprocess, sys

def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
            "lts__t_sectors_srcunit_tex_op_atom.sum", "l1tex__t_bytes.sum", "lts__t_bytes.sum"]
    idx = [h.index(c) if c in h else None for c in want]
    short = ["kernel", "us", "dramR", "dramW", "warps%", "regs", "stall_lsb", "stall_lgthr", "stall_bar", "stall_membar", "atom_sect", "l1B", "l2B"]
    print("\t".join(short))
    print("\t".join(rows[1][i] if i is not None else "-" for i in idx))
    for r in rows[2:]:
        vals = [r[i] if i is not None else "-" for i in idx]
        vals[0] = vals[0].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:34]
        print("\t".join(vals))

if __name__ == "__main__":
    main(sys.argv[1])
