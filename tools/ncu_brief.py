"""One-screen digest of an ncu --set full report: time, DRAM bytes, occupancy, issue, stall samples."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__occupancy_limit_warps",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static"]
STALLS = ["long_scoreboard", "barrier", "short_scoreboard", "lg_throttle", "mio_throttle", "wait", "selected",
          "not_selected", "math_pipe_throttle", "no_instruction", "branch_resolving", "dispatch_stall", "membar",
          "drain", "sleeping", "tex_throttle", "imc_miss", "misc"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, v = rows[0], rows[2]
    g = lambda k: v[h.index(k)] if k in h else "?"
    print("==", rep, g("Kernel Name")[:90])
    print("  " + "  ".join(f"{k.split('__')[1][:40]}={g(k)}" for k in KEYS))
    tot = float(g("smsp__pcsamp_sample_count"))
    st = {s: float(g("smsp__pcsamp_warps_issue_stalled_" + s)) for s in STALLS
          if g("smsp__pcsamp_warps_issue_stalled_" + s) != "?"}
    print("  stalls: " + "  ".join(f"{s} {100 * x / tot:.0f}%" for s, x in sorted(st.items(), key=lambda t: -t[1])[:7]))
