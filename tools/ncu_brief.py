"""Brief summary of one ncu --set full capture: duration, throughputs, stall mix, DRAM bytes.
  python tools/ncu_brief.py report.ncu-rep [kernel-regex]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
kf = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", f"regex:{kf}"] if kf else [])
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    def g(k):
        v = d.get(k, "")
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return None
    print(d.get("Kernel Name", "")[:60])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "smsp__inst_executed.sum",
              "sm__cycles_elapsed.avg.per_second"]:
        if k in d:
            print(f"  {k} = {d[k]} {units[hdr.index(k)]}")
    st = [(k, g(k)) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    st = [(k, v) for k, v in st if v]
    tot = sum(v for _, v in st) or 1
    print("  stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%"
                                   for k, v in sorted(st, key=lambda x: -x[1])[:8]))
