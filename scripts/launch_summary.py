"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel totals and shares."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        if "<" in name:
            name = name.split("<")[0] + "<" + name.split("<")[1].split(",")[0].split(">")[0] + ">"
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    out = [f"{'kernel':48s} {'launches':>8s} {'total_us':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k[:48]:48s} {cnt[k]:8d} {v / 1e3:10.1f} {v / allt * 100:6.1f}%")
    out.append(f"{'TOTAL':48s} {sum(cnt.values()):8d} {allt / 1e3:10.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(summarize(p))
