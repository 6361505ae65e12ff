"""Summarise an ncu report (``--set full``) into a short markdown table.

    python tools/ncu_summary.py gpurun_out/prof_hotspot.ncu-rep [--algo-bytes B] [--algo-flop F]

Reads ``ncu -i <rep> --page raw --csv`` (no GPU needed) and prints the
metrics the roofline accounting uses: duration, DRAM bytes (the
``traffic`` field of bench.py's roofline), throughputs, issue activity,
occupancy, registers and the top warp stall reasons.
"""

import argparse
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "instruction throughput %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "block limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "block limit (smem)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-instr"),
]


def raw(rep: str) -> list:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--algo-flop", type=float, default=None)
    a = ap.parse_args()
    for hdr, units, row in raw(a.rep):
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"### {d.get('Kernel Name', '?')}  grid {d.get('Grid Size', '')} block {d.get('Block Size', '')}")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in d:
                print(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = sorted(((float(v.replace(',', '')) if v.replace(',', '').replace('.', '', 1).isdigit() else 0.0, k)
                         for k, v in d.items()
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")),
                        reverse=True)[:6]
        if stalls:
            print("| top stalls (warps per issue) | " + ", ".join(
                f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
                for v, k in stalls) + " |")
        try:
            dur_ns = float(d["gpu__time_duration.sum"].replace(",", ""))
            unit = u.get("gpu__time_duration.sum", "ns")
            dur_s = dur_ns * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
                              "nsecond": 1e-9}.get(unit, 1e-9)
            rb = float(d["dram__bytes_read.sum"].replace(",", ""))
            wb = float(d["dram__bytes_write.sum"].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb *= scale.get(u.get("dram__bytes_read.sum", "byte"), 1)
            wb *= scale.get(u.get("dram__bytes_write.sum", "byte"), 1)
            print(f"| derived: DRAM traffic | {rb + wb:.4g} B ({(rb + wb) / dur_s / 1e9:.1f} GB/s) |")
            if a.algo_bytes:
                print(f"| derived: traffic / algorithmic bytes | {(rb + wb) / a.algo_bytes:.3f} |")
            if a.algo_flop:
                print(f"| derived: achieved FLOP/s | {a.algo_flop / dur_s / 1e12:.2f} TFLOP/s |")
        except (KeyError, ValueError):
            pass
        print()


if __name__ == "__main__":
    main()
