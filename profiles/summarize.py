"""Summarise ncu output into profiles/ (run here, on the files gpurun brought back).

    python profiles/summarize.py launches <launches.csv> <out.md>
    python profiles/summarize.py full <report.ncu-rep> <out.md>
    python profiles/summarize.py balance <kprof dir> <out.md>   (scripts/kprof.sh output)
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


def balance(d, out):
    """Per-kernel device time of one warm balance call per config phase."""
    import glob
    import os
    names = {"C3": ["vision", "audio", "llm"], "C4x30": ["vision", "audio", "llm"],
             "C4x64": ["vision", "audio", "llm"]}
    with open(out, "w") as f:
        f.write("# Balance kernels per launch\n\n`scripts/kprof.sh`: `ncu --profile-from-start off "
                "--metrics gpu__time_duration.sum --clock-control none` around the third (warm) "
                "`ctx.balance` call of each phase (cold-cache, serialised launches). C3 = DP=64 "
                "(single-CTA kernel), C4 = DP=2560 (30 and 64 examples per instance); vision and "
                "LLM phases GreedyUnpadded, audio BinaryPadded.\n\n")
        for path in sorted(glob.glob(os.path.join(d, "C*_[0-9].csv"))):
            cfg, ph = os.path.basename(path)[:-4].rsplit("_", 1)
            rows = list(csv.reader(open(path)))
            hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
            hdr = rows[hi]
            ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
            agg = collections.OrderedDict()
            for r in rows[hi + 1:]:
                k = r[ki].split("(")[0].replace("void ", "")
                k = k.split("::")[-1] if "orchb" in k else k[:60]
                a = agg.setdefault(k, [0, 0.0])
                a[0] += 1
                a[1] += float(r[vi].replace(",", ""))
            tot = sum(v for _, v in agg.values())
            n = sum(c for c, _ in agg.values())
            name = names.get(cfg, [ph] * 3)[int(ph)]
            f.write(f"## {cfg} {name}: {tot / 1e3:.1f} us device time over {n} launches\n\n"
                    "| us | launches | kernel |\n|---:|---:|---|\n")
            for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
                f.write(f"| {v / 1e3:.1f} | {c} | `{k}` |\n")
            f.write("\n")


if __name__ == "__main__":
    {"launches": launches, "full": full, "balance": balance}[sys.argv[1]](sys.argv[2], sys.argv[3])
