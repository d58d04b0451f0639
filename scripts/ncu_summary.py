"""Summarise an ncu report (raw page) into the numbers we track: duration, DRAM bytes and
throughput, occupancy, top stall reasons.  Usage: python scripts/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar_write_bytes.sum",
]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        out.append(f"kernel: {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k} = {vals[i]} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               h.startswith("smsp__pcsamp_warps_issue_stalled_"):
                try:
                    stalls.append((float(vals[i].replace(",", "")), h))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        for v, h in stalls[:8]:
            out.append(f"  stall {h} = {v}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(summarize(p))
