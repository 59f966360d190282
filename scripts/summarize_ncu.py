"""Summarise the ncu outputs of scripts/ncu_round.sh (in gpurun_out/) into profiles/:
  r01_ncu_launches_summary.csv   kernel share of a short bench run (serialised launch times)
  r01_ncu_vcycle_launches.csv    one V-cycle: per-launch time and DRAM bytes (warm caches)
  ncu_traffic.json               DRAM bytes per launch per bench kernel class (bench.py roofline)
  r01_ncu_full_<kernel>.json     selected metrics of the --set full captures"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
CLASS = [("k_cheb3_stream", "cheb0_fused"), ("k_chebM_stencil", "cheb0_fused"), ("k_cheb_stencil", "cheb0"), ("k_gcheb", "cheb_coarse"),
         ("k_acheb4", "cheb_coarse"), ("k_aresid4", "resid_coarse"), ("k_aspmv", "transfer"),
         ("k_gresid", "resid_coarse"), ("k_gspmv", "transfer"), ("k_resid_dinv_stencil", "resid0"),
         ("k_dense_gemv", "coarse_solve"), ("k_stencil_spmv", "spmv0"), ("k_multidot", "multidot"),
         ("k_multi_axpy_norm", "maxpy_norm"), ("k_assemble_had", "assemble"), ("k_delta_energy", "delta_energy")]


def klass(name):
    for k, c in CLASS:
        if k in name:
            return c
    return None


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    out = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = out.setdefault(r[h.index("ID")], {"name": r[h.index("Kernel Name")], "grid": r[h.index("Grid Size")]})
        d[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    return out


def short(name):
    return name.split("(")[0].replace("void ", "")


if os.path.exists(os.path.join(G, "launches.csv")):
    L = read_ncu_csv(os.path.join(G, "launches.csv"))
    agg = defaultdict(lambda: [0, 0.0, ""])
    for d in L.values():
        k = short(d["name"])
        agg[k][0] += 1
        agg[k][1] += d["gpu__time_duration.sum"] / 1e3
        agg[k][2] = d["grid"]
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(P, f"{TAG}_ncu_launches_summary.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "grid", "launches", "total_us", "us_per_launch", "share_pct"])
        for k, (n, us, g) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            w.writerow([k, g, n, round(us, 1), round(us / n, 2), round(100 * us / tot, 3)])
    print("launch list:", len(L), "launches")

traffic = {}
if os.path.exists(os.path.join(G, "vc_launches.csv")):
    V = read_ncu_csv(os.path.join(G, "vc_launches.csv"))
    per = defaultdict(lambda: [0, 0.0, 0.0])
    with open(os.path.join(P, f"{TAG}_ncu_vcycle_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "grid", "us", "dram_read_bytes", "dram_write_bytes", "l2_hit_pct"])
        for d in V.values():
            us = d["gpu__time_duration.sum"] / 1e3
            rb, wb = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
            w.writerow([short(d["name"]), d["grid"], round(us, 2), int(rb), int(wb),
                        round(d.get("lts__t_sector_hit_rate.pct", 0.0), 1)])
            c = klass(d["name"])
            if c:
                per[c][0] += 1
                per[c][1] += rb + wb
                per[c][2] += us
    # level-specific classes (bench.py's cheb_level1 / resid_level1 / transfer_level0): the level-1
    # launches are the k_acheb4 / k_aresid4 launches with the largest grid, the level-0 transfers
    # the k_aspmv launches with 2-row or 2-column blocks
    def gx(d):
        return int(d["grid"].strip("()").split(",")[0])
    for kname, cls in (("k_acheb4", "cheb_level1"), ("k_aresid4", "resid_level1")):
        ds = [d for d in V.values() if kname in d["name"]]
        if ds:
            g = max(gx(d) for d in ds)
            sel = [d for d in ds if gx(d) == g]
            per[cls] = [len(sel), sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
                                      for d in sel), 0.0]
    sel = [d for d in V.values() if "k_aspmv<4, 2" in d["name"] or "k_aspmv<2, 4" in d["name"]]
    if sel:
        per["transfer_level0"] = [len(sel), sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
                                                for d in sel), 0.0]
    for c, (n, b, us) in per.items():
        traffic[c] = b / n
    print("V-cycle launches:", len(V))


def full_metrics(rep, tag):
    if not os.path.exists(rep):
        return
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        return
    h = rows[0]
    keep = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
    units = rows[1]
    out = []
    for r in rows[2:]:
        out.append({k: (r[h.index(k)] + (" " + units[h.index(k)] if units[h.index(k)] else "")) for k in keep if k in h})
    json.dump(out, open(os.path.join(P, f"{TAG}_ncu_full_{tag}.json"), "w"), indent=1)
    print("full:", tag, len(out))


full_metrics(os.path.join(G, "prof_cheb3.ncu-rep"), "cheb0_fused")
full_metrics(os.path.join(G, "prof_gcheb.ncu-rep"), "gcheb_level1")
full_metrics(os.path.join(G, "prof_asm.ncu-rep"), "assemble")
full_metrics(os.path.join(G, "prof_krylov.ncu-rep"), "krylov")
# assembly / Krylov traffic from the full captures (bytes per launch)
for tag, cls in (("assemble", "assemble"),):
    fp = os.path.join(P, f"{TAG}_ncu_full_{tag}.json")
    if os.path.exists(fp):
        d = json.load(open(fp))[0]
        conv = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = d[k].split()
            tot += float(v) * conv[u]
        traffic[cls] = tot
if traffic:
    traffic["_source"] = (f"profiles/{TAG}_ncu_vcycle_launches.csv (one V-cycle, config 4 late iterate, warm "
                          f"caches) and profiles/{TAG}_ncu_full_assemble.json; DRAM bytes per launch, class mean")
    json.dump(traffic, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
    print("traffic:", {k: round(v / 1e6, 1) for k, v in traffic.items() if not k.startswith("_")}, "MB/launch")
