"""Per-CUDA-source-line hot spots of an ncu report (compile with -lineinfo): warp instructions
executed and stall samples, aggregated over every file the kernel's code comes from."""
import csv
import subprocess
import sys


def main(path, top=40, skip=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", str(skip)], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, recs = "?", []
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 8 or r[2] != "-":
            continue
        try:
            smp = int(r[4] or 0)
            ins = int(r[7] or 0)
        except ValueError:
            continue
        recs.append((ins, smp, f"{fname}:{r[0]}", r[1].strip()[:100]))
    ti = sum(x[0] for x in recs) or 1
    ts = sum(x[1] for x in recs) or 1
    print(f"warp instructions {ti:,}  stall samples {ts:,}")
    for ins, smp, loc, src in sorted(recs, reverse=True)[:top]:
        print(f"{100*ins/ti:5.1f}% inst {100*smp/ts:5.1f}% smp  {loc:18s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
