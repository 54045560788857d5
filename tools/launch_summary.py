"""Summarise an ncu --csv launch list: per-kernel count and total time for the
LAST step (from the last saso_plan_kernel launch to the end)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    ii = h.index("ID")
    out = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        out.setdefault(r[ii], [name, {}])[1][r[mi]] = float(r[vi].replace(",", ""))
    return list(out.values())


def main(path, start="saso_plan_kernel"):
    seq = load(path)
    idx = [i for i, (n, _) in enumerate(seq) if start in n]
    step = seq[idx[-1]:] if idx else seq
    agg = collections.OrderedDict()
    for n, m in step:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
    tot = sum(v for _, v in agg.values())
    for n, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n[:58]:58s} {c:4d} {v / 1e3:10.1f} us {100 * v / tot:5.1f}%")
    print(f"{'total':58s} {sum(c for c, _ in agg.values()):4d} {tot / 1e3:10.1f} us")
    ours = [(c, v) for n, (c, v) in agg.items() if n.startswith("cqg::")]
    print(f"{'ours (cqg::, excludes the harness setup kernels)':58s} {sum(c for c, _ in ours):4d} "
          f"{sum(v for _, v in ours) / 1e3:10.1f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
