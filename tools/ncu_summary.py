"""Summarise ncu outputs into small JSON files for profiles/ (development tool).

  python tools/ncu_summary.py launches <launches.csv> <out.json>
  python tools/ncu_summary.py full <report.ncu-rep | raw.csv> <out.json>
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
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    seq = []
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[mi].replace(",", "")) / 1e3   # ns -> us
        seq.append((name, v))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    res = {"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, "
           "serialised per-launch times; compare shares, not absolutes",
           "total_us": tot,
           "kernels": [{"kernel": k, "launches": v[0], "total_us": v[1], "share": v[1] / tot, "avg_us": v[1] / v[0]}
                       for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]}
    json.dump(res, open(out, "w"), indent=1)
    for k in res["kernels"][:12]:
        print(f"{k['kernel'][:40]:40s} {k['launches']:4d} {k['total_us']:10.1f} us {100 * k['share']:5.1f}%  avg {k['avg_us']:8.1f} us")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "launch__shared_mem_per_block_dynamic"]


WANT += ["lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
         "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full(path, out):
    if path.endswith(".csv"):                     # `ncu -i rep --page raw --csv` exported on the box
        txt = open(path).read()
    else:
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    res = {"source": path, "kernels": []}
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k in WANT:
            if k in h:
                i = h.index(k)
                d[k] = r[i] + ("" if not u[i] else " " + u[i])
        res["kernels"].append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res["kernels"]:
        print(json.dumps(d))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
