"""Summarise ncu captures for profiles/ (run HERE on the .ncu-rep files that
gpurun brought back; ncu -i works without a GPU).

  python tools/ncu_summary.py out.json name=gpurun_out/x.ncu-rep [name=...]
      -> per kernel launch: duration, DRAM bytes, throughput / pipe metrics
  python tools/ncu_summary.py --launches launches.csv out.csv
      -> per-kernel totals of an `ncu --metrics gpu__time_duration.sum,...
         --csv` launch list (share of the step, DRAM GB, GB/s)."""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = OrderedDict(kernel=r[hdr.index("Kernel Name")][:120])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = r[i] + (f" {units[i]}" if units[i] else "")
        res.append(d)
    return res


def launches(src, dst):
    rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iid = hdr.index("ID")
    per = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        key = (r[iid], r[ik])
        per.setdefault(key, {})[r[im]] = float(r[iv].replace(",", ""))
    agg = OrderedDict()
    for (_, name), m in per.items():
        a = agg.setdefault(name.split("(")[0], {"launches": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
        a["launches"] += 1
        a["ns"] += m.get("gpu__time_duration.sum", 0.0)
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["ns"] for a in agg.values())
    with open(dst, "w") as f:
        f.write(f"# total {tot / 1e3:.1f} us over {sum(a['launches'] for a in agg.values())} launches\n")
        f.write("kernel,launches,us,share,dram_read_GB,dram_write_GB,GBps\n")
        for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
            gbs = (a["rd"] + a["wr"]) / a["ns"] if a["ns"] else 0.0
            f.write(f"{name},{a['launches']},{a['ns'] / 1e3:.1f},{a['ns'] / tot:.3f},{a['rd'] / 1e9:.3f},"
                    f"{a['wr'] / 1e9:.3f},{gbs:.0f}\n")


def main():
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
        return
    out = OrderedDict()
    for spec in sys.argv[2:]:
        name, _, rep = spec.partition("=")
        out[name] = raw(rep)
    json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
