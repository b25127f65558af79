"""Counter evidence from an ncu report.

    python tools/ncu_counters.py REPORT.ncu-rep [--flops-per-launch F] [--label L]

Reads `ncu -i REPORT --page raw --csv` and prints, per profiled launch, the
executed FP32 / FP64 / tensor work from the SASS instruction counters, the
L2 and HBM bytes, the duration, and the derived achieved rates against the
B200 peaks (FP32 SIMT = SMs x 128 lanes x 2 x clock; FP64 = half of that;
HBM / 16-bit tensor = MEASURED_PEAKS.json), plus the top warp-stall reasons
and the shared-memory bank-conflict share.  JSON on stdout.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WANT = {
    "time_ns": "gpu__time_duration.sum",
    "ffma": "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "fadd": "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "fmul": "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "dfma": "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dadd": "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul": "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "lts_bytes": "lts__t_bytes.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
    "tensor_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "lds_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "lds_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "regs": "launch__registers_per_thread",
}
STALL_PREFIX = "smsp__pcsamp_warps_issue_stalled_"


def raw_rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units, data = rows[0], rows[1], rows[2:]
    return header, units, data


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarize(report, flops_per_launch=None, label=None):
    header, units, data = raw_rows(report)
    col = {h: i for i, h in enumerate(header)}
    peaks = {}
    ppath = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(ppath):
        peaks = json.load(open(ppath))
    out = []
    for row in data:
        g = {k: num(row[col[m]]) if m in col else None for k, m in WANT.items()}
        unit = {k: units[col[m]] for k, m in WANT.items() if m in col}
        # normalise: time to ns, bytes to bytes, clock to Hz
        if g["time_ns"] is not None:
            g["time_ns"] *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6,
                             "msecond": 1e6, "s": 1e9, "second": 1e9}.get(unit.get("time_ns"), 1)
        for b in ("lts_bytes", "dram_read", "dram_write"):
            u = unit.get(b, "byte")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            if g[b] is not None:
                g[b] *= scale
        if g["sm_clock_hz"] is not None:
            u = unit.get("sm_clock_hz", "hz")
            g["sm_clock_hz"] *= {"hz": 1, "Hz": 1, "Khz": 1e3, "Mhz": 1e6, "MHz": 1e6,
                                 "Ghz": 1e9, "GHz": 1e9}.get(u, 1)
        t = (g["time_ns"] or 0) / 1e9
        fp32 = 2 * (g["ffma"] or 0) + (g["fadd"] or 0) + (g["fmul"] or 0)
        fp64 = 2 * (g["dfma"] or 0) + (g["dadd"] or 0) + (g["dmul"] or 0)
        clk = g["sm_clock_hz"] or 1.965e9
        fp32_peak = 148 * 128 * 2 * clk
        rec = {
            "kernel": row[col["Kernel Name"]][:120] if "Kernel Name" in col else None,
            "label": label, "time_us": t * 1e6, "grid": g["grid"], "block": g["block"],
            "regs": g["regs"], "sm_clock_ghz": clk / 1e9,
            "fp32_executed_flop": fp32, "fp64_executed_flop": fp64,
            "fp32_tflops": fp32 / t / 1e12 if t else None,
            "fp32_frac_of_simt_peak": fp32 / t / fp32_peak if t else None,
            "fp64_tflops": fp64 / t / 1e12 if t else None,
            "fp64_frac_of_peak": fp64 / t / (fp32_peak / 2) if t else None,
            "l2_bytes": g["lts_bytes"], "l2_gbs": g["lts_bytes"] / t / 1e9 if t and g["lts_bytes"] else None,
            "dram_bytes": (g["dram_read"] or 0) + (g["dram_write"] or 0),
            "dram_gbs": ((g["dram_read"] or 0) + (g["dram_write"] or 0)) / t / 1e9 if t else None,
            "dram_frac_of_measured": (((g["dram_read"] or 0) + (g["dram_write"] or 0)) / t / 1e9
                                      / peaks["hbm_gbs"]) if t and "hbm_gbs" in peaks else None,
            "tensor_pipe_active_pct": g["tensor_active_pct"], "fma_pipe_active_pct": g["fma_pipe_pct"],
            "fp64_pipe_active_pct": g["fp64_pipe_pct"], "issue_active_pct": g["issue_active_pct"],
            "shared_ld_wavefronts": g["lds_wavefronts"], "shared_ld_bank_conflicts": g["lds_conflicts"],
            "shared_ld_conflict_share": (g["lds_conflicts"] / g["lds_wavefronts"])
            if g["lds_wavefronts"] and g["lds_conflicts"] is not None else None,
        }
        if flops_per_launch:
            rec["algorithmic_flop"] = flops_per_launch
            rec["algorithmic_tflops"] = flops_per_launch / t / 1e12 if t else None
        stalls = {}
        for h, i in col.items():
            if h.startswith(STALL_PREFIX) and "not_issued" not in h and "." not in h:
                v = num(row[i])
                if v:
                    stalls[h[len(STALL_PREFIX):]] = v
        tot = sum(stalls.values())
        if tot:
            rec["stall_share_top"] = {k: round(v / tot, 3) for k, v in
                                      sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--flops-per-launch", type=float, default=None)
    ap.add_argument("--label", default=None)
    a = ap.parse_args()
    json.dump(summarize(a.report, a.flops_per_launch, a.label), sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
