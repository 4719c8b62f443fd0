"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

  python tools/launch_summary.py gpurun_out/launches_r01.csv "command line" > profiles/r01_launches_summary.txt
"""
import collections
import csv
import sys


def main(path, cmd):
    rows = list(csv.reader(open(path)))
    i = [j for j, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, body = rows[i], rows[i + 1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt, units = collections.Counter(), collections.Counter(), set()
    for r in body:
        name = r[ik].split("(")[0].replace("void ", "").replace("gtcp::", "")
        tot[name] += float(r[iv].replace(",", ""))
        cnt[name] += 1
        units.add(r[iu])
    allt = sum(tot.values())
    print(f"# ncu launch list of `{cmd}` (1 B200)")
    print(f"# metric gpu__time_duration.sum, --clock-control none; cold-cache serialised: compare SHARES. units: {units}")
    print(f"# {len(body)} launches\n")
    print(f"{'kernel':45s} {'launches':>8s} {'total':>14s} {'share':>7s} {'avg':>12s}")
    for k, v in tot.most_common():
        print(f"{k[:45]:45s} {cnt[k]:8d} {v:14.0f} {100 * v / allt:6.1f}% {v / cnt[k]:12.0f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
