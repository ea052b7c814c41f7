"""Summarise an ncu --set full report: per-launch duration, DRAM bytes, tensor-pipe and
throughput percentages (reads `ncu -i <rep> --page raw --csv`)."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "name": "Kernel Name", "grid": "Grid Size", "block": "Block Size",
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_B": "dram__bytes_read.sum", "dram_write_B": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "tc_inst_pct": "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread", "smem_B": "launch__shared_mem_per_block_dynamic",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    col = {}
    for k, m in METRICS.items():
        for i, name in enumerate(h):
            if name == m or name.endswith("." + m) or name.split(".", 2)[-1] == m:
                col[k] = i
                break
    out = []
    for r in rows[2:]:
        d = {}
        for k, i in col.items():
            v = r[i]
            try:
                v = float(v.replace(",", ""))
                u = units[i]
                if u in ("Kbyte", "KB"):
                    v *= 1e3
                elif u in ("Mbyte", "MB"):
                    v *= 1e6
                elif u in ("Gbyte", "GB"):
                    v *= 1e9
                elif u in ("usecond", "us"):
                    v *= 1e3
                elif u in ("msecond", "ms"):
                    v *= 1e6
            except ValueError:
                pass
            d[k] = v
        out.append(d)
    return out


if __name__ == "__main__":
    res = {rep: summarize(rep) for rep in sys.argv[1:]}
    print(json.dumps(res, indent=1))
