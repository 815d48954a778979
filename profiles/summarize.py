"""Summarise ncu output into profiles/ (run here, on the files gpurun brought back).

    python profiles/summarize.py launches <launches.csv> <out.md>
    python profiles/summarize.py full <report.ncu-rep> <out.md>
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0][:80]
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v for _, v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({path})\n\n`gpu__time_duration.sum`, --clock-control none; "
                "cold-cache, serialised launches: compare shares, not absolutes.\n\n")
        f.write("| launches | total us | share | kernel |\n|---:|---:|---:|---|\n")
        for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| {c} | {v / 1e3:.1f} | {100 * v / tot:.1f}% | `{k}` |\n")
        f.write(f"\ntotal {tot / 1e3:.1f} us over {sum(c for c, _ in agg.values())} launches\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "smsp__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({path})\n\n")
        for r in rows[2:]:
            f.write(f"## `{r[hdr.index('Kernel Name')][:100]}`\n\n| metric | value | unit |\n|---|---:|---|\n")
            for w in WANT:
                if w in hdr:
                    i = hdr.index(w)
                    f.write(f"| {w} | {r[i]} | {units[i]} |\n")
            if "dram__bytes_read.sum" in hdr:
                def val(name):
                    i = hdr.index(name)
                    x = float(r[i].replace(",", ""))
                    u = units[i]
                    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
                traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
                f.write(f"| traffic (read+write) | {traffic:.0f} | byte |\n")
            f.write("\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
