"""Shared-memory wavefronts per CUDA source line (actual vs ideal) of an ncu report's source page.
Usage: python tools/ncu_wavefronts.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, hdr, cur = [], None, None
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
    d = dict(zip(hdr, r))
    if d.get("Address", "-") != "-":   # SASS rows: the CUDA rows carry the per-line totals
        continue
    try:
        wf = float(d.get("L1 Wavefronts Shared", "0") or 0)
        wi = float(d.get("L1 Wavefronts Shared Ideal", "0") or 0)
        ins = float(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    if wf > 0:
        rows.append((wf, wi, ins, f"{cur}:{r[0]}", d.get("Source", "")[:90]))
tot = sum(x[0] for x in rows)
print(f"total shared wavefronts {tot:.4g}")
for wf, wi, ins, loc, src in sorted(rows, reverse=True)[:15]:
    print(f"{100 * wf / tot:5.1f}%  wf {wf:.3g} ideal {wi:.3g}  ({wf / max(ins, 1):.2f}/instr)  {loc}  {src}")
