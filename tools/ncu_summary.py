"""Summarise an ncu report (raw page) into the metrics we track per kernel."""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_us"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed", "fma_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed", "alu_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed", "lsu_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefront_pct"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_elapsed", "issue_pct"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_inst_pct"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_inst_pct"),
    ("dram__bytes_read.sum", "dram_read_bytes"),
    ("dram__bytes_write.sum", "dram_write_bytes"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "registers"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall_math_throttle"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_short_sb"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall_dispatch"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall_mio"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall_not_selected"),
]


def summarise(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    # bytes -> bytes; durations -> microseconds (ncu prints "us"/"ms"/"ns")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        rec = {"kernel": re.sub(r"\(.*", "", d.get("Kernel Name", "?"))[:60]}
        for k, name in KEYS:
            if k in d:
                try:
                    v = float(d[k].replace(",", ""))
                    v *= scale.get(units.get(k, ""), 1)
                    rec[name] = v
                except ValueError:
                    rec[name] = d[k]
        out.append(rec)
    return out


if __name__ == "__main__":
    import json
    for rep in sys.argv[1:]:
        for rec in summarise(rep):
            print(json.dumps(rec))
