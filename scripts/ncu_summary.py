"""Key metrics of an ncu --set full report, one block per profiled launch.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep > profiles/rNN_x_ncu_summary.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (HMMA) active %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (tcgen05) active %"),
    ("sm__inst_executed_pipe_tc.sum", "tcgen05 instructions"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "warp cycles per issued instruction"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    unit = dict(zip(hdr, units))
    print(f"# ncu --set full summary of {path.split('/')[-1]} ({len(data)} launches; serialised, cold unless noted)")
    for r in data:
        d = dict(zip(hdr, r))
        print(f"\n## {d.get('Kernel Name', '?')[:90]}")
        for k, label in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                print(f"  {label:40s} {d[k]} {unit.get(k, '')}")
        stalls = sorted(((float(d[k]), k) for k in hdr if "warps_issue_stalled" in k and
                         k.endswith("per_issue_active.ratio") and d.get(k) not in ("", "n/a", None)), reverse=True)[:5]
        print("  top stalls (warps per issue): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, k in stalls))


if __name__ == "__main__":
    main(sys.argv[1])
