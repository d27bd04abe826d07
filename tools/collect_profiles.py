"""Copy one round_profiles.sh run (gpurun_out/<tag>) into tracked summaries under profiles/ (<prefix>_*).
Usage: python tools/collect_profiles.py gpurun_out/r1b r1b"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(path):
    try:
        lines = [l for l in open(path).read().strip().splitlines() if l.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = []
    for v in rows[2:]:
        d = dict(zip(rows[0], v))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in d:
                try:
                    d[k] = float(d[k].replace(",", "")) * scale.get(rows[1][rows[0].index(k)], 1.0)
                except ValueError:
                    pass
        res.append(d)
    return res


def main(src, prefix):
    prof = os.path.join(ROOT, "profiles")
    for name in ["default", "c1", "c2", "c3", "c4", "c5"]:
        d = last_json(os.path.join(src, f"bench_{name}.log"))
        if d:
            json.dump(d, open(os.path.join(prof, f"{prefix}_bench_{name}.json"), "w"), indent=1)
    for f in ["launches_c4.txt", "launches_c4.csv"]:
        p = os.path.join(src, f)
        if os.path.exists(p):
            open(os.path.join(prof, f"{prefix}_{f}"), "w").write(open(p).read())
    with open(os.path.join(prof, f"{prefix}_gpu_tests.txt"), "w") as o:
        for f in ["env.txt", "smoke.log", "tests.log"]:
            p = os.path.join(src, f)
            if os.path.exists(p):
                o.write(f"# {f}\n" + "".join(open(p).readlines()[-40:]) + "\n")
    traffic = {}
    with open(os.path.join(prof, f"{prefix}_ncu_summary.txt"), "w") as o:
        o.write(f"# ncu --set full --clock-control none summaries ({prefix}); per-line hot spots from tools/ncu_lines.py\n")
        for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep")):
            path = os.path.join(src, rep)
            o.write(f"\n#### {rep}\n")
            o.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), path],
                                   capture_output=True, text=True).stdout)
            o.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), path, "12"],
                                   capture_output=True, text=True).stdout)
            for d in raw(path):
                try:
                    rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
                except (KeyError, ValueError):
                    continue
                traffic[rep[:-8]] = {"kernel": d.get("Kernel Name", "")[:60], "dram_read_bytes": rd,
                                     "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                                     "ncu_duration": d.get("gpu__time_duration.sum", "")}
    json.dump(traffic, open(os.path.join(prof, f"{prefix}_ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
