"""Key metrics of an ncu --set full report (one kernel): time, DRAM bytes, throughputs, stalls."""
import csv
import re
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
keys = re.compile(r"^(Kernel Name|gpu__time_duration.sum|dram__bytes_read.sum|dram__bytes_write.sum|"
                  r"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|dram__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"lts__throughput.avg.pct_of_peak_sustained_elapsed|sm__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"lts__t_sector_hit_rate.pct|launch__registers_per_thread|launch__grid_size|"
                  r"launch__shared_mem_per_block_dynamic|sm__warps_active.avg.pct_of_peak_sustained_active|"
                  r"lts__t_sectors_srcunit_tex_op_read.sum|lts__t_sectors_srcunit_tex_op_atom.sum|"
                  r"smsp__inst_executed.sum|l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum|"
                  r"smsp__pcsamp_warps_issue_stalled_[a-z_]+)$")
for v in rows[2:]:
    for i, n in enumerate(h):
        if keys.match(n) and v[i] not in ("", "0"):
            print("%-70s %-12s %s" % (n, u[i], v[i]))
    print("-" * 100)
