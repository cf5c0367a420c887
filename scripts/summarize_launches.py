"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > iv:
            try:
                agg[r[ik].split("(")[0].replace("void ", "")].append(float(r[iv].replace(",", "")))
            except ValueError:
                pass
    tot = sum(sum(v) for v in agg.values())
    print(f"| kernel | launches | total us | share | mean us |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {100*sum(v)/tot:.1f}% | {sum(v)/len(v)/1e3:.2f} |")


if __name__ == "__main__":
    main(sys.argv[1])
