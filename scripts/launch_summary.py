"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys


def summarise(path, title):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    skip = ("init_slab", "elementwise", "vectorized", "distribution", "reduce_kernel", "Fill", "fill")
    tot = sum(v[1] for k, v in agg.items() if not any(s in k for s in skip))
    out = [f"### {title}\n", "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        sh = "" if any(s in k for s in skip) else f"{t / tot:.1%}"
        out.append(f"| {k} | {n} | {t / 1e3:.1f} | {sh} | {t / n / 1e3:.1f} |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print(summarise(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]))
