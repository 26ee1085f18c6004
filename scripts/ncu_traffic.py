"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant
kernels from `ncu --set full` reports into profiles/ncu_traffic.json, which bench.py reads for
the roofline `traffic` field.

    python scripts/ncu_traffic.py --k2 mixtral=gpurun_out/k2_mix.ncu-rep qwen3=... \
        --k2-bytes mixtral=704660000 ... --gemm mixtral_prefill=gpurun_out/pf.ncu-rep

Each entry records the captured launch's DRAM bytes and its algorithmic bytes (K2: rows x 6d +
activations, from scripts/k2_bench.py's k2_MB), so bench.py can report traffic per launch as
(DRAM / algorithmic) x its own algorithmic bytes per launch.
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dram_bytes(path, kernel_substr):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ik = hdr.index("Kernel Name")
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = []
    for r in data:
        if kernel_substr in r[ik]:
            b = float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]]
            res.append((r[ik], b))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k2", nargs="*", default=[], help="config=report")
    ap.add_argument("--k2-bytes", nargs="*", default=[], help="config=algorithmic bytes of the captured launch")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
    a = ap.parse_args()
    alg = dict(x.split("=") for x in a.k2_bytes)
    db = json.load(open(a.out)) if os.path.exists(a.out) else {}
    for item in a.k2:
        cfg, path = item.split("=")
        launches = dram_bytes(path, "k2_split_expert")
        if not launches:
            continue
        dram = sum(b for _, b in launches) / len(launches)
        ent = {"kernel": "k2_split_expert", "report": os.path.relpath(path, ROOT), "dram_bytes_per_launch": dram,
               "launches_captured": len(launches)}
        if cfg in alg:
            ent["alg_bytes_per_launch"] = float(alg[cfg])
            ent["ratio"] = dram / float(alg[cfg])
        db[cfg] = ent
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(db, open(a.out, "w"), indent=1)
    print(json.dumps(db, indent=1))


if __name__ == "__main__":
    main()
