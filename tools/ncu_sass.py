"""Per-SASS-instruction hot spots of an ncu report (ncu -i --page source --csv --print-source sass).
Usage: python tools/ncu_sass.py report.ncu-rep [top]  -> top instructions by stall samples, and
shared-memory instructions with excessive wavefronts (bank conflicts)."""
import csv
import io
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    body = rows[1:]

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError, IndexError):
            return 0.0
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in body) or 1.0
    print(f"{len(body)} SASS lines, {tot:.0f} samples")
    hot = sorted(body, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]
    for r in hot:
        print(f"{100 * f(r, 'Warp Stall Sampling (All Samples)') / tot:5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:70]}")
    print("-- shared memory: excessive wavefronts")
    sm = sorted(body, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:12]
    for r in sm:
        if f(r, "L1 Wavefronts Shared Excessive") > 0:
            print(f"  excess {f(r, 'L1 Wavefronts Shared Excessive'):.3g} of {f(r, 'L1 Wavefronts Shared'):.3g}  "
                  f"{r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:60]}")
    # instruction mix
    mix = {}
    for r in body:
        op = r[ix["Source"]].strip().split(" ")[0]
        if op.startswith("@"):
            op = r[ix["Source"]].strip().split(" ")[1]
        op = op.split(".")[0]
        mix[op] = mix.get(op, 0) + f(r, "Instructions Executed")
    t = sum(mix.values()) or 1.0
    print("-- instruction mix (warp-level executed)")
    print("  " + ", ".join(f"{k} {100 * v / t:.1f}%" for k, v in sorted(mix.items(), key=lambda x: -x[1])[:16]))
    print(f"  total warp instructions {t:.4g}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
