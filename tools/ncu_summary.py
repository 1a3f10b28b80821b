"""Summarise an ncu report (raw page) into the numbers the roofline needs.

    python tools/ncu_summary.py gpurun_out/prof_cfg2.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    # memory-system view (round 2, session 4): LSU data pipe, SM -> XBAR write port, L2 slices, cross-die sectors
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed", "l1tex__m_l1tex2xbar_write_bytes.sum.per_second",
    "l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors.sum.per_second", "lts__t_sectors_srcunit_tex.sum.per_second",
    "lts__t_sectors_srcunit_ltcfabric.sum.per_second", "lts__t_sector_hit_rate.pct",
    "dram__bytes.sum.per_second",
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.3:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res.append(d)
    return res


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    txt = json.dumps(res, indent=1)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            f.write(txt + "\n")
    print(txt)
