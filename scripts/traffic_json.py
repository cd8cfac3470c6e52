"""Per-launch DRAM traffic table for bench.py from exported ncu raw CSVs.

    python scripts/traffic_json.py OUT.json ITER_RAW.csv.gz DAS_RAW.csv.gz CFG5_RAW.csv.gz TAG

ITER_RAW: one cfg3 iteration (--set full); DAS_RAW: the cfg3 DAS kernel;
CFG5_RAW: one cfg5 iteration.  Kernel names are shortened the way ncu prints
them without the namespace."""
import csv
import gzip
import json
import re
import sys

DAS_KEYS = ["smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "gpu__time_duration.sum"]


UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
UNITS = {}


def rows(path):
    r = list(csv.reader(gzip.open(path, "rt") if path.endswith(".gz") else open(path)))
    hdr = r[0]
    UNITS[path] = dict(zip(hdr, r[1]))
    return [dict(zip(hdr, x), _path=path) for x in r[2:] if len(x) == len(hdr)]


def short(name):
    n = re.sub(r"\(.*", "", name)
    n = n.replace("unnamed>::", "").replace("void ", "").strip()
    return n


def traffic(path):
    out = {}
    for d in rows(path):
        k = short(d["Kernel Name"])
        if k in out:
            continue  # first launch of each kernel
        try:
            out[k] = int(float(d["dram__bytes_read.sum"]) * scale(d, "dram__bytes_read.sum") +
                         float(d["dram__bytes_write.sum"]) * scale(d, "dram__bytes_write.sum"))
        except (KeyError, ValueError):
            pass
    return out


def scale(d, key):  # the unit row of the --page raw --csv export
    return UNIT.get(UNITS[d["_path"]].get(key, "byte"), 1.0)


def main():
    out_path, it, das, c5, tag = sys.argv[1:6]
    t = {"_source": f"ncu --set full --clock-control none (scripts/gpu_profiles.sh, {tag}); "
                    "dram__bytes_read.sum + dram__bytes_write.sum per launch, first launch of each kernel"}
    t.update(traffic(it))
    t["_cfg5"] = traffic(c5)
    d = [r for r in rows(das) if "das_stack" in r["Kernel Name"]][0]
    t["_das_cfg3"] = {k: float(d[k]) for k in DAS_KEYS if k in d}
    json.dump(t, open(out_path, "w"), indent=1)
    print(json.dumps({k: v for k, v in t.items() if not k.startswith("_")}, indent=1))


if __name__ == "__main__":
    main()
