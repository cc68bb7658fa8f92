"""Condense an `ncu --set full` capture of tools/profile_step.py into the
per-kernel JSON summary committed under profiles/ (bench.py reads the
enclose kernel's DRAM traffic from it).

    python tools/make_ncu_summary.py REPORT.ncu-rep OUT.json [capture-command]

Per kernel (first launch of each name): duration, DRAM bytes read/written,
registers, fp64-pipe / issue activity, executed DP flops, top stall reasons,
and the achieved fraction of the measured HBM / fp64 peaks.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
STALLS = ["math_pipe_throttle", "wait", "not_selected", "short_scoreboard", "long_scoreboard",
          "dispatch_stall", "branch_resolving", "lg_throttle", "mio_throttle", "barrier",
          "membar", "no_instruction", "drain", "selected"]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def val(h, units, r, key, scale=True):
    if key not in h:
        return None
    i = h.index(key)
    try:
        x = float(r[i].replace(",", ""))
    except ValueError:
        return None
    return x * UNIT.get(units[i], 1.0) if scale else x


def short(name):
    base = name.split("(")[0].replace("void ", "").strip()
    return base.split("::")[-1]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    capture = sys.argv[3] if len(sys.argv) > 3 else None
    h, units, rows = load(rep)
    peaks = {}
    mp = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    if mp.exists():
        peaks = json.loads(mp.read_text())
    kernels = {}
    for r in rows:
        name = r[h.index("Kernel Name")]
        key = short(name)
        if key in kernels:
            continue
        t = val(h, units, r, "gpu__time_duration.sum")
        rd = val(h, units, r, "dram__bytes_read.sum")
        wr = val(h, units, r, "dram__bytes_write.sum")
        cyc = val(h, units, r, "sm__cycles_elapsed.avg.per_second", scale=False)
        k = {"kernel": name[:160], "duration_ms": t * 1e3 if t else None,
             "dram_read_bytes": rd, "dram_write_bytes": wr,
             "dram_bytes": (rd or 0) + (wr or 0),
             "registers_per_thread": val(h, units, r, "launch__registers_per_thread", False),
             "warps_active_pct": val(h, units, r,
                                     "sm__warps_active.avg.pct_of_peak_sustained_active", False),
             "issue_active_pct": val(h, units, r,
                                     "sm__issue_active.avg.pct_of_peak_sustained_elapsed", False),
             "fp64_pipe_active_pct": val(
                 h, units, r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 False)}
        if t:
            k["dram_gbs"] = k["dram_bytes"] / t / 1e9
            if peaks.get("hbm_gbs"):
                k["dram_frac_of_measured_hbm"] = k["dram_gbs"] / peaks["hbm_gbs"]
        # executed DP flops = per-cycle rates x elapsed cycles (DFMA counts 2)
        dp = 0.0
        inst = {}
        cycles = val(h, units, r, "sm__cycles_elapsed.avg", False)
        for op, w in (("dfma", 2), ("dmul", 1), ("dadd", 1)):
            x = val(h, units, r,
                    f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed",
                    False)
            if x is not None and cycles:
                dp += w * x * cycles
                inst[op] = x * cycles  # thread instructions per launch
        if dp:
            k["executed_dp_flops"] = dp
            k["executed_dp_thread_inst"] = inst
            if t:
                k["executed_dp_tflops"] = dp / t / 1e12
        st = []
        for s in STALLS:
            x = val(h, units, r, f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio",
                    False)
            if x:
                st.append((s, round(x, 3)))
        k["stall_top"] = [f"{a} {b}" for a, b in sorted(st, key=lambda z: -z[1])[:5]]
        if cyc:
            k["sm_clock_ghz"] = cyc
        kernels[key] = k
    doc = {"capture": capture, "report": Path(rep).name, "kernels": kernels}
    Path(out).write_text(json.dumps(doc, indent=1) + "\n")
    for key, k in kernels.items():
        print(f"{key:28s} {k['duration_ms'] or 0:9.3f} ms  dram {k['dram_bytes'] / 1e6:9.1f} MB")


if __name__ == "__main__":
    main()
