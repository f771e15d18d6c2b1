"""Summarize an ncu --set full report of pass kernels (profiles/ format):
python tools/ncu_summary.py gpurun_out/prof_pass_C2.ncu-rep "C2" m n l"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "launch__grid_size", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]


def main():
    rep, name = sys.argv[1], sys.argv[2]
    m, n, l = (int(x) for x in sys.argv[3:6])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    alg = 8.0 * (m * n + n * l + m * l) / 1e9
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")]
        kind = "apply" if "pass_kernel<1" in kname else "adjoint"
        print(f"## {name} {kind}: {kname[:70]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:100s} {r[i]} {units[i]}")
        rd = float(r[hdr.index("dram__bytes_read.sum")])
        wr = float(r[hdr.index("dram__bytes_write.sum")])
        ur = units[hdr.index("dram__bytes_read.sum")]
        scale = {"Mbyte": 1e-3, "Gbyte": 1.0, "Kbyte": 1e-6, "byte": 1e-9}.get(ur, 1.0)
        tr = (rd + wr * ({"Mbyte": 1e-3, "Gbyte": 1.0, "Kbyte": 1e-6}.get(units[hdr.index("dram__bytes_write.sum")], 1.0) / scale)) * scale
        print(f"  traffic (read+write) = {tr:.4f} GB; algorithmic = {alg:.4f} GB; ratio {tr / alg:.3f}\n")


if __name__ == "__main__":
    main()
