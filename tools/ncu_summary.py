"""Summaries of ncu output for profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launch-list.csv>      per-kernel time shares
  python tools/ncu_summary.py full <report.ncu-rep> [...]      key --set full metrics

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


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2:])
