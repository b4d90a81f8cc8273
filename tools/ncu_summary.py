"""Summarise ncu outputs into committed files under profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.md>
      per-kernel launch count, total / average device time and DRAM bytes
      (from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,...`)
  python tools/ncu_summary.py full <report.ncu-rep> <out.json>
      key `--set full` metrics per profiled kernel (duration, DRAM bytes,
      L2 hit rate, achieved occupancy, top stall reasons)
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, mi, ii = (h.index("Kernel Name"), h.index("Metric Value"),
                      h.index("Metric Name"), h.index("ID"))
    per = collections.defaultdict(lambda: collections.defaultdict(dict))
    for r in rows[hi + 1:]:
        if len(r) > vi:
            per[r[ki].split("(")[0]][r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    lines = ["| kernel | launches | total us | avg us | share | DRAM MB/launch |",
             "|---|---|---|---|---|---|"]
    tot_all = sum(m.get("gpu__time_duration.sum", 0) for k in per.values() for m in k.values())
    for k, ls in sorted(per.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1].values())):
        t = [m.get("gpu__time_duration.sum", 0) for m in ls.values()]
        d = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in ls.values()]
        lines.append(f"| `{k}` | {len(t)} | {sum(t)/1e3:.1f} | {sum(t)/len(t)/1e3:.2f} | "
                     f"{sum(t)/max(tot_all,1):.1%} | {sum(d)/len(d)/1e6:.2f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "launch__grid_size",
            "launch__registers_per_thread", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum"]
    res = []
    for r in rows[2:]:
        e = {"kernel": r[h.index("Kernel Name")].split("(")[0], "id": r[h.index("ID")]}
        for k in keys:
            if k in h:
                try:
                    e[k] = float(r[h.index(k)].replace(",", ""))
                except ValueError:
                    e[k] = r[h.index(k)]
                e[k + ".unit"] = u[h.index(k)]
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        e["top_stalls"] = [s for _, s in sorted(st, reverse=True)[:5]]
        res.append(e)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(path, workload, out="profiles/ncu_traffic.json"):
    """Merge per-kernel DRAM bytes per launch (read + write, averaged over the
    captured launches of each kernel) of one `--set full` report into
    profiles/ncu_traffic.json under `workload` (bench.py reads it for the
    roofline `traffic` field)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    per = collections.defaultdict(list)
    for r in rows[2:]:
        k = r[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").replace("fae::", "").strip()
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[h.index(m)].replace(",", "")) * _SCALE[u[h.index(m)]]
        per[k].append(b)
    try:
        cur = json.load(open(out))
    except Exception:
        cur = {}
    w = cur.setdefault(workload, {})
    for k, v in per.items():
        w[k] = {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v), "report": path.split("/")[-1]}
    json.dump(cur, open(out, "w"), indent=1)
    print(json.dumps(cur, indent=1))


def traffic_launches(path, workload, out="profiles/ncu_traffic.json"):
    """Same as `traffic`, from a launch list (`--metrics gpu__time_duration.sum,
    dram__bytes_read.sum,dram__bytes_write.sum`: one pass per launch, no
    kernel replay, so the caches hold what the real run left in them;
    averaged over every captured launch of each kernel)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, mi, ii, ui = (h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"),
                          h.index("ID"), h.index("Metric Unit"))
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi].startswith("dram__bytes"):
            k = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("fae::", "").strip()
            per[k][r[ii]] += float(r[vi].replace(",", "")) * _SCALE.get(r[ui], 1.0)
    try:
        cur = json.load(open(out))
    except Exception:
        cur = {}
    w = cur.setdefault(workload, {})
    for k, v in per.items():
        w[k] = {"dram_bytes_per_launch": sum(v.values()) / len(v), "launches": len(v),
                "source": path.split("/")[-1] + " (launch list, no replay)"}
    json.dump(cur, open(out, "w"), indent=1)
    print(json.dumps(cur, indent=1)[:1500])


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic, "traffic_launches": traffic_launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
