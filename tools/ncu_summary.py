"""Summarise an ncu --set full report into the metrics DESIGN.md / profiles/ cite.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--bytes-model B] > profiles/x.txt

Runs here (no GPU): `ncu -i <rep> --page raw --csv`.  One block per profiled
launch: duration, DRAM bytes, L1TEX / LTS sector counts, occupancy, issue
activity and the top warp stall reasons.
"""
import argparse
import csv
import io
import subprocess

KEYS = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "L1 global ld requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global ld sectors"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit %"),
    ("l1tex__data_pipe_lsu_wavefronts.sum", "L1 data-pipe wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "LTS sectors read (from SM)"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "LTS throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--bytes-model", type=float, default=None,
                    help="algorithmic bytes per launch (reports DRAM / model)")
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        print("---")
        rd = wr = None
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"{label:32s} {r[i]} {units[i]}")
                if key == "dram__bytes_read.sum":
                    rd = (r[i], units[i])
                if key == "dram__bytes_write.sum":
                    wr = (r[i], units[i])
        if args.bytes_model and rd and wr:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = float(rd[0]) * scale[rd[1]] + float(wr[0]) * scale[wr[1]]
            print(f"{'DRAM bytes / model bytes':32s} {tot / args.bytes_model:.3f}")
        stalls = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:6]
        for v, h in stalls:
            name = h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
            print(f"{'stall ' + name:32s} {v:.2f} per issue")


if __name__ == "__main__":
    main()
