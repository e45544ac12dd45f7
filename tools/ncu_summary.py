"""Summarise gpurun_out ncu artefacts into profiles/ (tracked evidence).

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of a run
    python tools/ncu_summary.py full <prof.ncu-rep> [regex]         # key counters per launch

Prints markdown; `--json out.json` also writes the numbers.
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("lts__t_sectors.sum", "l2_bytes"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "sector": 32.0}


def short(name):
    m = re.match(r"(?:void )?(?:pdhg::)?([\w]+)(<[^()]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", "nsecond"), 1e-9)
                k = short(d["Kernel Name"])
                agg[k][0] += 1
                agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": n, "total_ms": t * 1e3, "mean_us": t / n * 1e6, "share": t / tot})
    return out


def full(path, regex=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if regex and not re.search(regex, name):
            continue
        d = {"kernel": short(name)}
        for key, alias in KEYS:
            if key in hdr:
                i = hdr.index(key)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[alias] = v * SCALE.get(units[i], 1.0)
        out.append(d)
    return out


def main():
    mode, path = sys.argv[1], sys.argv[2]
    js = None
    if "--json" in sys.argv:
        js = sys.argv[sys.argv.index("--json") + 1]
    rest = [a for a in sys.argv[3:] if a != "--json" and a != js]
    if mode == "launches":
        res = launches(path)
        print("| kernel | launches | total ms | mean us | share |\n|---|---|---|---|---|")
        for d in res[:20]:
            print(f"| `{d['kernel']}` | {d['launches']} | {d['total_ms']:.2f} | {d['mean_us']:.2f} | {100 * d['share']:.1f}% |")
    else:
        res = full(path, rest[0] if rest else None)
        print("| kernel | us | DRAM rd MB | DRAM wr MB | L2 MB | DRAM % | SM % | L2 hit % | occ % | regs |\n"
              "|---|---|---|---|---|---|---|---|---|---|")
        for d in res:
            print(f"| `{d['kernel']}` | {d.get('time', 0) * 1e6:.1f} | {d.get('dram_rd', 0) / 1e6:.2f} | "
                  f"{d.get('dram_wr', 0) / 1e6:.2f} | {d.get('l2_bytes', 0) / 1e6:.2f} | {d.get('dram_pct', 0):.1f} | "
                  f"{d.get('sm_pct', 0):.1f} | {d.get('l2_hit_pct', 0):.1f} | {d.get('occupancy_pct', 0):.1f} | "
                  f"{d.get('regs', 0):.0f} |")
    if js:
        json.dump(res, open(js, "w"), indent=1)


if __name__ == "__main__":
    main()
