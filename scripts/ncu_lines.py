"""Per-source-line hot spots of an ncu report (needs -lineinfo): instructions executed and stall samples."""
import csv
import subprocess
import sys


def main(path, top=40, kernel=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda"]
    if kernel:
        cmd += ["-k", kernel]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    recs = []
    for r in rows:
        if len(r) > 3 and r[0] in ("#", "Line"):
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                recs.append((int(d.get("Warp Stall Sampling (All Samples)", 0) or 0),
                             int(d.get("Instructions Executed", 0) or 0), d.get("#", d.get("Line", "")),
                             d.get("Source", "")[:110]))
            except ValueError:
                pass
    tot_s = sum(r[0] for r in recs) or 1
    tot_i = sum(r[1] for r in recs) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for s, i, ln, src in sorted(recs, reverse=True)[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  L{ln:>5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else None)
