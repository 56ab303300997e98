"""Summaries of ncu exports for profiles/ (tuning aid, run here on the CSVs
gpurun brings back):

    python tools/ncu_summaries.py launches <launches.csv[.gz]> <out.json> "<command>"
        per-kernel launch count / average / share of the gpu__time_duration
        launch list (ncu serialises launches and runs them cold: compare
        shares, not totals).  The persistent frame loop is a cooperative
        cluster launch that ncu cannot replay, so the list is taken with it
        excluded (-k regex:'^(?!.*frame_loop)'); its time comes from the bench
        line's CUDA-event `kernels` table instead (merged when --bench is given).
    python tools/ncu_summaries.py traffic <raw.csv[.gz]> <out.json>
        per kernel category (gemm = hoisted NT GEMMs, dw = grouped dW):
        DRAM bytes, tensor-pipe activity, L2 hit rate and L2->SM bytes per
        launch, averaged over the captured launches of that kind.
"""
from __future__ import annotations

import csv
import gzip
import json
import sys
from collections import defaultdict


def _open(path):
    return gzip.open(path, "rt") if path.endswith(".gz") else open(path)


def _rows(path):
    rows = list(csv.reader(_open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            return r, rows[i + 1:]
    raise SystemExit(f"{path}: no ncu header")


def launches(path, out, command, bench=None):
    hdr, rows = _rows(path)
    ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if len(r) <= vi or not r[vi]:
            continue
        key = f"{r[ki]} grid {r[gi]}"
        agg[key][0] += 1
        agg[key][1] += float(r[vi].replace(",", ""))
    total = sum(v[1] for v in agg.values())
    kern = [{"kernel": k, "launches": n, "avg_ns": t / n, "share": t / total}
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    res = {"command": command,
           "note": "ncu serialises launches and flushes caches (cold): compare shares, not totals; the "
                   "persistent frame loop (cooperative cluster launch, not replayable under ncu) is excluded "
                   "from the list -- see frame_loop_from_bench",
           "unit": "ns", "launches": sum(v[0] for v in agg.values()), "kernels": kern}
    if bench:
        line = json.loads(open(bench).read().strip().splitlines()[-1])
        ks = line.get("kernels", {})
        step = line["ms_per_step"]
        res["frame_loop_from_bench"] = {
            "source": bench, "ms_per_step": step,
            "categories": {k: {"ms_per_step": v["ms_per_step"], "launches_per_step": v["launches_per_step"],
                               "share_of_step": v["ms_per_step"] / step} for k, v in ks.items()}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(kern[:8], indent=1))


def _category(name):
    if "tma_frame_loop" in name:
        return "gemm_frame"
    if "tma_gemm_persistent" in name and "DwGroup" in name:
        return "dw"
    if "tma_gemm_persistent" in name or "tma_gemm_kernel" in name:
        return "gemm"
    return None


def traffic(path, out):
    rows = list(csv.reader(_open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        v = r[col[name]].replace(",", "")
        try:
            return float(v)
        except ValueError:  # "", "n/a", "no data"
            return 0.0

    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "%": 1.0}
    tensor = next((h for h in hdr if h.endswith("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")),
                  None)
    def get(r, name):
        return val(r, name) * scale.get(units[col[name]], 1.0)

    acc = defaultdict(lambda: defaultdict(float))
    names, count = {}, defaultdict(int)
    for r in data:
        cat = _category(r[col["Kernel Name"]])
        if cat is None:
            continue
        names[cat] = r[col["Kernel Name"]]
        count[cat] += 1
        a = acc[cat]
        a["dram_read_bytes"] += get(r, "dram__bytes_read.sum")
        a["dram_write_bytes"] += get(r, "dram__bytes_write.sum")
        a["duration_us"] += get(r, "gpu__time_duration.sum")
        a["tensor_pipe_active_pct"] += val(r, tensor) if tensor else 0.0
        a["tmem_tensor_active_pct"] += val(r, "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        a["l2_hit_pct"] += val(r, "lts__t_sector_hit_rate.pct")
        a["l2_to_sm_bytes"] += get(r, "lts__t_sectors_srcunit_tex.sum") * 32 if "lts__t_sectors_srcunit_tex.sum" in col \
            else 0.0
    res = {}
    for cat, a in acc.items():
        n = count[cat]
        d = {k: v / n for k, v in a.items()}
        d["dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        d["kernel"] = names[cat]
        d["launches_averaged"] = n
        res[cat] = d
    old = {}
    try:
        old = json.load(open(out))
    except (OSError, ValueError):
        pass
    for k, v in old.items():
        if k not in res and k != "gemm_frame":
            res[k] = v  # keep categories this capture did not cover
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else None)
    else:
        traffic(sys.argv[2], sys.argv[3])
