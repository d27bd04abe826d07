"""Stall samples and executed instructions per CUDA source line of an ncu report.
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr = None, None
    agg, ins, txt = collections.Counter(), collections.Counter(), {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        try:
            ln = int(r[0])
            s, n = float(r[4] or 0), float(r[7] or 0)
        except (ValueError, IndexError):
            continue
        agg[(cur, ln)] += s
        ins[(cur, ln)] += n
        txt[(cur, ln)] = r[1]
    tot, tn = sum(agg.values()) or 1.0, sum(ins.values()) or 1.0
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}% stall  {100 * ins[k] / tn:5.1f}% inst  {k[0]}:{k[1]}  {txt[k].strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
