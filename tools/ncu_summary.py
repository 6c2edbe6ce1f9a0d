"""Summarise ncu artefacts into profiles/<round>_ncu_summary.json (+ .md).

    python tools/ncu_summary.py --round r01 --launches gpurun_out/launches_r01.csv \
        --rep adamw=gpurun_out/prof_adamw.ncu-rep --rep pack=gpurun_out/prof_pack.ncu-rep

* launch list (``--metrics gpu__time_duration.sum``): per-kernel launch count,
  total / mean device time and SHARE of the listed time (cold-cache,
  serialised: compare shares, not absolutes);
* ``--set full`` captures: per launch dram bytes read+write (the roofline
  "traffic"), duration, registers, occupancy, and the algorithmic bytes of
  the same launch derived from the kernel's arguments (28 B/elem AdamW,
  4 B/elem bf16 pack) so traffic/algorithmic shows re-reads.
"""

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OURS = re.compile(r"hod::|pack_kernel|adamw_vec_kernel|adamw_scalar_kernel|sumsq_kernel|p2p_step_kernel|span_tma_kernel|"
                  r"barrier_kernel|norm_exchange_kernel|sum_partials_kernel|clip_coef_kernel|pack_adamw|pack_sumsq|"
                  r"accumulate_partials")


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)(<[^(]*>)?", name)
    if not m:
        return name[:60]
    return (m.group(1) + (m.group(2) or "")).replace("unsigned short", "bf16")


def launches(path: Path) -> dict:
    text = path.read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit] * v
        k = short(r["Kernel Name"])
        per[k][0] += 1
        per[k][1] += us
        total += us
    ours_total = sum(t for k, (n, t) in per.items() if OURS.search(k))
    out = {k: {"launches": n, "total_us": round(t, 2), "mean_us": round(t / n, 3),
               "share_of_listed": round(t / total, 4), "ours": bool(OURS.search(k)),
               "share_of_ours": round(t / ours_total, 4) if OURS.search(k) else None}
           for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}
    return {"kernels": out, "listed_total_us": round(total, 2), "ours_total_us": round(ours_total, 2)}


def rep(path: Path, bytes_per_elem_read: float, bytes_per_elem_write: float, elem_from: str) -> dict:
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        v = float(r[col[name]].replace(",", ""))
        u = units[col[name]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
                 "msecond": 1e3}.get(u, 1)
        return v * scale

    launches_ = []
    for r in rows[2:]:
        rd = val(r, "dram__bytes_read.sum")
        wr = val(r, "dram__bytes_write.sum")
        us = val(r, "gpu__time_duration.sum")
        launches_.append({
            "kernel": short(r[col["Kernel Name"]]),
            "duration_us": round(us, 3),
            "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
            "dram_GBps": round((rd + wr) / us / 1e3, 1),
            "dram_pct_peak": float(r[col["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]]),
            "registers": int(float(r[col["launch__registers_per_thread"]])),
            "grid": int(float(r[col["launch__grid_size"]])),
            "warps_active_pct": float(r[col["sm__warps_active.avg.pct_of_peak_sustained_active"]]),
            "sm_throughput_pct": float(r[col["sm__throughput.avg.pct_of_peak_sustained_elapsed"]]),
        })
    # algorithmic bytes: element count inferred from the dominant streamed input
    for L in launches_:
        n = L["dram_read_bytes"] / bytes_per_elem_read if elem_from == "read" else None
        L["elements_inferred"] = int(round(n)) if n else None
    return {"launches": launches_}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[], help="name=path.ncu-rep")
    ap.add_argument("--note", default="")
    ap.add_argument("--each", help="path.ncu-rep of tools/ncu_each.py (one launch per kernel)")
    ap.add_argument("--each-order", help="tools/ncu_each.py stdout (launch order + algorithmic bytes)")
    ap.add_argument("--out-dir", default=str(ROOT / "profiles"))
    a = ap.parse_args()
    if a.each:
        line = next(x for x in reversed(Path(a.each_order).read_text().splitlines())
                    if x.startswith('{"launch_order"'))   # ncu interleaves its ==PROF== lines
        order = json.loads(line)["launch_order"]
        r = rep(Path(a.each), 1, 1, "none")["launches"]
        if len(r) != len(order):
            raise SystemExit(f"{len(r)} profiled launches vs {len(order)} in the launch order")
        doc = {"round": a.round, "note": a.note, "kernels": {}}
        for L, o in zip(r, order):
            L.pop("elements_inferred", None)
            tr = L["dram_read_bytes"] + L["dram_write_bytes"]
            L.update({"elements": o.get("elems") or o.get("owned_elems"), "algorithmic_bytes": o["algorithmic_bytes"],
                      "traffic_over_algorithmic": round(tr / o["algorithmic_bytes"], 3),
                      "algorithmic_GBps": round(o["algorithmic_bytes"] / L["duration_us"] / 1e3, 1)})
            doc["kernels"][o["name"]] = L
        out = Path(a.out_dir) / f"{a.round}_ncu_each.json"
        out.write_text(json.dumps(doc, indent=1) + "\n")
        print(out)
        return
    doc = {"round": a.round, "note": a.note, "kernels": {}}
    if a.launches:
        doc["launch_list"] = launches(Path(a.launches))
    spec = {"adamw": (14, 14, 28), "pack": (2, 2, 4), "pack_adamw": (14, 14, 28), "fused": (None, None, 28),
            "pack_sumsq": (2, None, 2), "fused_emulated_d2": (None, None, None)}
    for item in a.rep:
        name, path = item.split("=", 1)
        rd, wr, alg = spec.get(name, (None, None, None))
        r = rep(Path(path), rd or 1, wr or 1, "read" if rd else "none")
        per_launch = []
        for L in r["launches"]:
            n = L["elements_inferred"]
            L["algorithmic_bytes"] = alg * n if (alg and n) else None
            L["traffic_over_algorithmic"] = (round((L["dram_read_bytes"] + L["dram_write_bytes"]) /
                                                   L["algorithmic_bytes"], 3) if L["algorithmic_bytes"] else None)
            per_launch.append(L)
        mean_traffic = sum(L["dram_read_bytes"] + L["dram_write_bytes"] for L in per_launch) / len(per_launch)
        mean_alg = (sum(L["algorithmic_bytes"] for L in per_launch) / len(per_launch)
                    if all(L["algorithmic_bytes"] for L in per_launch) else None)
        doc["kernels"][name] = {"source": Path(path).name, "launches": per_launch,
                                "dram_bytes_per_launch": int(mean_traffic),
                                "algorithmic_bytes_per_launch": int(mean_alg) if mean_alg else None}
    out = Path(a.out_dir) / f"{a.round}_ncu_summary.json"
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(doc, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
