"""Summarise ncu reports into profiles/ (run here, on the CPU box, after a gpurun).

usage: python scripts/ncu_summary.py TAG   (reads gpurun_out/prof_{fwd,bwd}_TAG.ncu-rep,
        gpurun_out/launches_TAG.csv; writes profiles/TAG_*.csv and updates
        profiles/ncu_summary.json, which bench.py reads for roofline.traffic)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "gpc__cycles_elapsed.avg.per_second"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows


def main(tag):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ.setdefault("dram_bytes_per_launch", {})
    summ.setdefault("rounds", {})
    rnd = {}
    for k in ("fwd", "bwd", "fwd0", "bwd0", "mask"):
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{k}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        rows = raw(rep)
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = {}
        for key in KEYS:
            if key in hdr:
                i = hdr.index(key)
                d[key] = {"value": vals[i], "unit": units[i]}
        rb = float(d["dram__bytes_read.sum"]["value"]) * UNIT.get(d["dram__bytes_read.sum"]["unit"], 1)
        wb = float(d["dram__bytes_write.sum"]["value"]) * UNIT.get(d["dram__bytes_write.sum"]["unit"], 1)
        d["dram_bytes_total"] = rb + wb
        name = {"fwd": "fmha_fwd", "bwd": "fmha_bwd", "fwd0": "fmha_fwd_p0", "bwd0": "fmha_bwd_p0",
                "mask": "dropout_mask"}[k]
        rnd[name] = d
        summ["dram_bytes_per_launch"][name] = rb + wb
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{k}_raw.csv"), "w") as f:
            csv.writer(f).writerows(rows)
    # HBM-bound gather kernels (a5 / a6 / a9): one metrics row per launch
    gp = os.path.join(ROOT, "gpurun_out", f"gather_{tag}.csv")
    if os.path.exists(gp):
        lines = [l for l in open(gp) if not l.startswith("==")]
        rows = list(csv.reader(io.StringIO("".join(lines))))
        hdr = rows[0]
        ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        per = {}
        idi = hdr.index("ID")
        for r in rows[1:]:
            if len(r) <= vi:
                continue
            v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
            per.setdefault((r[idi], r[ki][:60]), {})[r[mi]] = v
        out = []
        for (lid, k), m in per.items():
            t = m.get("gpu__time_duration.sum", 0.0)
            by = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            out.append({"kernel": k, "us": round(t * 1e6, 2), "dram_bytes": by,
                        "dram_GBps": round(by / t / 1e9, 1) if t else None})
        with open(os.path.join(ROOT, "profiles", f"{tag}_gather_ncu.json"), "w") as f:
            json.dump(out, f, indent=1)
        rnd["gather"] = f"profiles/{tag}_gather_ncu.json"
        for e in out:
            summ["dram_bytes_per_launch"].setdefault("gather", {})[e["kernel"]] = e["dram_bytes"]
    lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(lp):
        lines = [l for l in open(lp) if not l.startswith("==")]
        rows = list(csv.reader(io.StringIO("".join(lines))))
        hdr = rows[0]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        launches = [{"kernel": r[ki][:90], "time": r[vi], "unit": r[ui]} for r in rows[1:] if len(r) > vi]
        with open(os.path.join(ROOT, "profiles", f"{tag}_launches.json"), "w") as f:
            json.dump(launches, f, indent=1)
        rnd["launch_list"] = f"profiles/{tag}_launches.json"
    summ["rounds"][tag] = rnd
    summ["note"] = ("ncu --set full --clock-control none, one launch of each FMHA main kernel from "
                    "scripts/probe_time.py (config 2 batch; fmha_fwd / fmha_bwd at p = 0.1 with the "
                    "materialised keep bits -- the headline -- and *_p0 at p = 0 from r02c on); dram bytes "
                    "are per launch")
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(rnd, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
