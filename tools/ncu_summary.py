"""Key raw metrics of every kernel in an ncu report (usage: ncu_summary.py REPORT)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
STALLS = "smsp__average_warps_issue_stalled_"
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:90])
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"   {k:70s} {r[i]:>16} {units[i]}")
    st = [(float(r[i]), h[len(STALLS):].replace("_per_issue_active.ratio", ""))
          for i, h in enumerate(hdr) if h.startswith(STALLS) and h.endswith("per_issue_active.ratio")
          and r[i] not in ("", "n/a")]
    st.sort(reverse=True)
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:7]))
