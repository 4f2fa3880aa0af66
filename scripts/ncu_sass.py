"""SASS-level summary of an ncu report: instruction mix by opcode and the hottest instructions by stall samples."""
import collections
import csv
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix_src, ix_s, ix_i = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    ops = collections.Counter()
    smp = collections.Counter()
    lines = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        src = r[ix_src].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        base = op.split(".")[0]
        try:
            n, s = int(r[ix_i] or 0), int(r[ix_s] or 0)
        except ValueError:
            continue
        ops[base] += n
        smp[base] += s
        lines.append((s, n, r[0], src))
    ti, ts = sum(ops.values()) or 1, sum(smp.values()) or 1
    print(f"warp instructions {ti:,}  stall samples {ts:,}")
    for op, n in ops.most_common(25):
        print(f"  {op:10s} {100*n/ti:5.1f}% inst  {100*smp[op]/ts:5.1f}% samples")
    print("hottest instructions:")
    for s, n, addr, src in sorted(lines, reverse=True)[:top]:
        print(f"  {100*s/ts:5.1f}% {n:>12,} {addr[-5:]} {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
