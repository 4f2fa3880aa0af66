"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel count and total ms,
and the per-generation shares (the last `--per` launches form one generation if given)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")[:70]
        v = float(r["Metric Value"])
        unit = r.get("Metric Unit", "ns")
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        tot[name] += ms
        cnt[name] += 1
    T = sum(tot.values()) or 1
    print(f"{len(rows)} launches, {T:.3f} ms total (serialised, cold-cache)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:9.3f} ms {100*v/T:5.1f}%  x{cnt[k]:<5d} {k}")


if __name__ == "__main__":
    main(sys.argv[1])
