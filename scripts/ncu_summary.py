"""Summarise an ncu --set full report (raw page) into the metrics the roofline uses."""
import csv
import io
import re
import subprocess
import sys

PAT = re.compile(r"^(gpu__time_duration.sum|dram__bytes_read.sum|dram__bytes_write.sum|"
                 r"sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed|"
                 r"sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed|"
                 r"sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"lts__throughput.avg.pct_of_peak_sustained_elapsed|"
                 r"dram__throughput.avg.pct_of_peak_sustained_elapsed|"
                 r"sm__cycles_elapsed.avg.per_second|launch__registers_per_thread|"
                 r"launch__grid_size|launch__cluster_dim_x|sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed|"
                 r"sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed|"
                 r"lts__t_sector_hit_rate.pct|smsp__inst_executed.sum)$")


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:80]
        print(f"## {name}")
        for i, k in enumerate(h):
            if PAT.match(k):
                print(f"  {k} = {r[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
