"""Record the DRAM traffic of kernels from an `ncu --set full` capture into profiles/traffic.json,
with the hash of the CUDA sources the capture was taken on (bench.py reports `roofline.traffic`
only when that hash matches the sources it benchmarks).

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep [more.ncu-rep ...]

Per kernel class (bench.py's names): dram__bytes_read.sum + dram__bytes_write.sum per launch,
averaged over the captured launches of that kernel."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import TRAFFIC_JSON, src_hash  # noqa: E402

CLASS_OF = {"k_cg_matvec_pull_p": "cg_dist", "k_cg_matvec_pull": "cg_dist", "k_rhs_pull": "rhs", "k_cg_matvec_tma": "cg_dist", "k_rhs_tma": "rhs", "k_cg_update4": "cg_update",
            "k_dist_project1": "dist_project", "k_dist_first": "dist_first", "k_dist_replay1": "dist_replay", "k_predict": "predict",
            "k_wave_project": "dist_project", "k_wave_replay": "dist_replay", "k_cg_tetv": "cg_tet",
            "k_tet_psd": "tet_replay"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def kernel_class(name):
    for k, c in CLASS_OF.items():
        if k in name:
            return c, k
    return None, None


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    res = {}
    for r in data:
        cls, short = kernel_class(r[col["Kernel Name"]])
        if not cls:
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[col[m]].replace(",", "")) * UNIT.get(units[col[m]], 1.0)
        dur = float(r[col["gpu__time_duration.sum"]].replace(",", "")) if "gpu__time_duration.sum" in col else None
        e = res.setdefault(cls, {"kernel": short, "bytes": [], "us": []})
        e["bytes"].append(b)
        if dur is not None:
            e["us"].append(dur * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(units[col["gpu__time_duration.sum"]], 1.0))
    return res


def main():
    kern = {}
    for rep in sys.argv[1:]:
        for cls, e in read(rep).items():
            kern[cls] = {"kernel": e["kernel"], "dram_bytes_per_launch": sum(e["bytes"]) / len(e["bytes"]),
                         "launches_captured": len(e["bytes"]),
                         "ncu_duration_us": (sum(e["us"]) / len(e["us"])) if e["us"] else None, "capture": rep}
    d = {"src_sha": src_hash(), "capture": ", ".join(os.path.relpath(r, ROOT) for r in sys.argv[1:]), "kernels": kern}
    json.dump(d, open(TRAFFIC_JSON, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
