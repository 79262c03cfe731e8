"""Build profiles/ncu_summary.json from an `ncu --set full` capture of the N=1
bench (read with `ncu -i ... --page raw --csv`).

    python scripts/ncu_summarize.py gpurun_out/prof_n1.ncu-rep [N]

Per kernel: duration, DRAM bytes read/written per launch, the algorithmic
bytes of one launch and the achieved fraction of the
measured copy peak in MEASURED_PEAKS.json.  bench.py reads
`kernels[<key>].dram_bytes_per_launch` for `roofline.traffic`.
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "launch__registers_per_thread",
           "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
        "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def algorithmic_bytes(kernel: str, n: int) -> tuple[str, int]:
    if "ec_direct_step_kernel" in kernel:
        return "direct_step", 16 * n          # read x, w; write u, w
    if "ec_update_gen_kernel" in kernel:
        return "update", 12 * n               # read u, w; write w
    if "ec_direct_round" in kernel:
        return "round_p1", 8 * n
    if "ec_fold_auto_kernel" in kernel:
        return "fold", 0                      # zero-copy offer: posts only
    return kernel.split("(")[0].split()[-1], 0


def main(rep: str, n: int = 25_559_081) -> None:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    kernels = {}
    for r in data:
        rec = dict(zip(head, r))
        u = dict(zip(head, units))

        def val(m):
            return float(rec[m].replace(",", "")) * UNIT.get(u[m], 1)

        name = rec["Kernel Name"]
        key, alg = algorithmic_bytes(name, n)
        dur = val("gpu__time_duration.sum")
        k = {"kernel": name.split("(")[0], "duration_us": dur,
             "dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum"),
             "registers": int(val("launch__registers_per_thread")),
             "grid": int(val("launch__grid_size")),
             "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
             "algorithmic_bytes": alg}
        k["dram_bytes_per_launch"] = k["dram_read"] + k["dram_write"]
        if alg:
            k["algorithmic_gbs"] = alg / (dur * 1e-6) / 1e9
            k["frac_of_measured_peak"] = k["algorithmic_gbs"] / peak
        kernels.setdefault(key, k)
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    # merge: entries of kernels this capture does not launch (e.g. the P>1
    # update kernel, captured earlier) are kept with their own source note
    old = {}
    if os.path.exists(path):
        with open(path) as f:
            old = json.load(f).get("kernels", {})
    src = os.path.basename(rep)
    for k in kernels.values():
        k["capture"] = src
    merged = {**old, **kernels}
    summary = {"source": "ncu --set full --clock-control none of the N=1 bench; one launch per "
                         "kernel after warm-up; cold-cache, serialised (per-entry `capture`)",
               "n_elems": n, "measured_peak_gbs": peak, "kernels": merged}
    with open(path, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:]))
