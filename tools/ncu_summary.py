"""Summaries of ncu output for profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launch-list.csv>      per-kernel time shares
  python tools/ncu_summary.py full <report.ncu-rep> [...]      key --set full metrics
  python tools/ncu_summary.py quick <metrics.csv>              tools/ncu_quick.sh output: per kernel, last launch
  python tools/ncu_summary.py traffic <report.ncu-rep> [...]   DRAM bytes per launch -> JSON
                                                               (profiles/ncu_traffic.json, read by bench.py)

The launch list comes from
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file F \
      python bench.py --profile --steps 1 --warmup 3
(cold-cache, serialised launches: compare SHARES with bench.py's stage times,
not absolute durations).
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    per = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "").strip()
        ns = float(r[14].replace(",", ""))
        c, t = per.get(name, (0, 0.0))
        per[name] = (c + 1, t + ns)
    total = sum(t for _, t in per.values())
    print(f"launch list: {path} ({len(rows)} launches, {total / 1e6:.3f} ms total)\n")
    print("| kernel | launches | total ms | mean us/launch | share |")
    print("|---|---:|---:|---:|---:|")
    for name, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {c} | {t / 1e6:.3f} | {t / c / 1e3:.1f} | {100 * t / total:.1f}% |")


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def quick(path):
    """Per kernel (the last launch of each name): the targeted metric set."""
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    cols = rows[hdr]
    ci = {c: i for i, c in enumerate(cols)}
    per = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) != len(cols):
            continue
        name = r[ci["Kernel Name"]].split("(")[0].replace("void ", "").strip()
        per.setdefault((name, int(r[ci["ID"]])), {})[r[ci["Metric Name"]]] = (r[ci["Metric Value"]], r[ci["Metric Unit"]])
    last = collections.OrderedDict()
    for (name, lid), m in per.items():
        last[name] = m
    for name, m in last.items():
        print(f"### `{name}`\n")
        print("| metric | value | unit |\n|---|---:|---|")
        for k in sorted(m):
            print(f"| `{k}` | {m[k][0]} | {m[k][1]} |")
        print()


def full(paths):
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rd = csv.reader(io.StringIO(out))
        hdr = next(rd)
        units = next(rd)
        for vals in rd:
            d = dict(zip(hdr, vals))
            u = dict(zip(hdr, units))
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
            print(f"### `{name}` ({path})\n")
            print("| metric | value |")
            print("|---|---:|")
            for k, label in KEYS:
                if k in d:
                    print(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
            st = []
            for k, x in d.items():
                if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                    try:
                        st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x.replace(",", ""))))
                    except ValueError:
                        pass
            tot = sum(x for _, x in st) or 1.0
            st.sort(key=lambda t: -t[1])
            print("\nwarp-stall samples: " + ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in st[:6]) + "\n")


# bench.py stage -> kernels whose DRAM traffic makes up the stage
STAGE_KERNELS = {
    "border.prefilter": ["k_border_prefilter"],
    "border.scan32": ["k_border_scan32"],
    "border.exact": ["k_border_exact"],
    "border.wide": ["k_border_wide"],
    "border.infinite": ["k_border_infinite"],
    "border.grid": ["k_owner_mark", "k_field_tiles"],
    "assign.table": ["k_vlt_build"],
    "assign.points": ["k_assign_vlt", "k_assign_overflow"],
}


def traffic_quick(path):
    """tools/ncu_quick.sh output -> per kernel (largest launch, the step's main
    one) DRAM bytes and warp instructions, per bench stage: the JSON bench.py
    reads (profiles/ncu_traffic.json)."""
    import json
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = {k: i for i, k in enumerate(rows[0])}
    per = {}
    for r in rows[1:]:
        if r[0] == "ID":
            continue
        name = r[h["Kernel Name"]].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
        key = (name, r[h["ID"]])
        per.setdefault(key, {})[r[h["Metric Name"]]] = float(r[h["Metric Value"]].replace(",", ""))
    best = {}
    for (name, _), m in per.items():
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        t = m.get("gpu__time_duration.sum", 0.0)
        if name not in best or t > best[name]["ns"]:
            best[name] = {"dram_bytes": b, "inst": m.get("smsp__inst_executed.sum", 0.0), "ns": t}
    res = {"source": [path], "kernels": best, "stages": {}, "inst": {}}
    for st, ks in STAGE_KERNELS.items():
        if all(k in best for k in ks):
            res["stages"][st] = sum(best[k]["dram_bytes"] for k in ks)
            res["inst"][st] = sum(best[k]["inst"] for k in ks)
    print(json.dumps(res, indent=1))


def traffic(paths):
    import json
    per = {}
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rd = csv.reader(io.StringIO(out))
        hdr = next(rd)
        units = next(rd)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        for vals in rd:
            d = dict(zip(hdr, vals))
            u = dict(zip(hdr, units))
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
            b = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                b += float(d[k].replace(",", "")) * scale.get(u.get(k, "byte"), 1)
            per.setdefault(name, []).append(b)
    res = {"source": [str(p) for p in paths], "kernels": {k: sum(v) / len(v) for k, v in per.items()}, "stages": {}}
    for st, ks in STAGE_KERNELS.items():
        if all(k in res["kernels"] for k in ks):
            res["stages"][st] = sum(res["kernels"][k] for k in ks)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2:])
    elif sys.argv[1] == "quick":
        quick(sys.argv[2])
    elif sys.argv[1] == "traffic_quick":
        traffic_quick(sys.argv[2])
    else:
        full(sys.argv[2:])
