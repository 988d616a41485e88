#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv>      # per-kernel counts, device time, share
  python tools/ncu_summary.py full <prof.ncu-rep> [...]     # key metrics of a --set full capture
  python tools/ncu_summary.py traffic <workload> <sketch.ncu-rep> <longpass.ncu-rep>   # -> profiles/traffic.json
  python tools/ncu_summary.py dram <launches.csv>          # per-kernel DRAM bytes of a launch list
"""
import collections
import csv
import json
import re
import subprocess
import sys

OURS = ("sketch_dense_kernel", "sketch_finish_kernel", "sketch_csr", "csr_", "rowpass_kernel", "colreduce_kernel",
        "lsqr_", "fill_kernel", "copy_scale_kernel", "transpose_kernel", "extract_r_kernel", "form_nt_kernel",
        "debug_gaussian", "bulk_", "lsrn")


def short(name):
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"^void ", "", n)
    n = re.sub(r"<.*", "", n) if not n.startswith(("sketch_dense", "rowpass")) else n
    return n.split("::")[-1][:80]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.OrderedDict()
    total = ours_total = 0.0
    for r in rows[i + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        t = float(r[mv].replace(",", "")) / 1e3   # ns -> us
        nm = short(r[kn])
        mine = any(o in r[kn] for o in OURS)
        a = agg.setdefault(nm, {"count": 0, "us": 0.0, "ours": mine})
        a["count"] += 1
        a["us"] += t
        total += t
        ours_total += t if mine else 0.0
    out = []
    for nm, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        out.append({"kernel": nm, "ours": a["ours"], "launches": a["count"], "total_us": round(a["us"], 1),
                    "avg_us": round(a["us"] / a["count"], 2), "share_of_all": round(a["us"] / total, 4)})
    return {"total_us": round(total, 1), "ours_us": round(ours_total, 1), "kernels": out}


def dram(path):
    """Per kernel of a launch list with dram__bytes_read.sum / dram__bytes_write.sum: launches,
    total and average DRAM bytes (read + write) and device time."""
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    kn, mv, mn, idc = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) <= mv:
            continue
        d = per.setdefault(r[idc], {"name": short(r[kn])})
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else ""
        v = float(r[mv].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        d[r[mn]] = v * scale
    agg = collections.OrderedDict()
    for d in per.values():
        a = agg.setdefault(d["name"], {"launches": 0, "dram_bytes": 0.0, "ns": 0.0})
        a["launches"] += 1
        a["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a["ns"] += d.get("gpu__time_duration.sum", 0.0)
    return {nm: {"launches": a["launches"], "dram_bytes": a["dram_bytes"], "avg_dram_bytes": a["dram_bytes"] / a["launches"],
                 "total_us": a["ns"] / 1e3} for nm, a in agg.items()}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        res.append(d)
    return res


def traffic(workload, sketch_rep, lp_rep, out="profiles/traffic.json"):
    """Record dram read+write bytes per launch of the sketch and long-pass kernels."""
    def bytes_of(rep, kernel_re):
        for d in full(rep):
            if re.search(kernel_re, d["kernel"]):
                tot = 0.0
                for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v, unit = d[key].split()
                    tot += float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
                return tot
        return None
    try:
        cur = json.load(open(out))
    except Exception:
        cur = {}
    cur[workload] = {"sketch": bytes_of(sketch_rep, "sketch"), "long_pass": bytes_of(lp_rep, "rowpass|csr_rowdot"),
                     "source": f"ncu --set full: {sketch_rep}, {lp_rep}"}
    json.dump(cur, open(out, "w"), indent=1)
    return cur


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    elif mode == "traffic":
        print(json.dumps(traffic(sys.argv[2], sys.argv[3], sys.argv[4]), indent=1))
    elif mode == "dram":
        print(json.dumps(dram(sys.argv[2]), indent=1))
    else:
        print(json.dumps([full(p) for p in sys.argv[2:]], indent=1))
