"""Write profiles/traffic_<config>.json from an `ncu --set full` capture: DRAM
bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of each kernel
of the fast-scan stage (A3-A6) and their sum, which bench.py reports as the
roofline `traffic` of that stage.

  python tools/traffic_from_ncu.py <report.ncu-rep|.csv> <config> [out.json] [searches] [scan_path] [nprobe]

`searches` = number of searches the report covers (default 1: an NVTX-filtered
capture of one search, `tools/profile_step.py` + `ncu --nvtx --nvtx-include
"search/"`); per-search bytes = the stage kernels' total / searches (a search
may launch a kernel more than once, e.g. the selection in query halves).
"""
import csv
import json
import subprocess
import sys

STAGE = ("lut_tiles_kernel", "lm_count_kernel", "lm_scan_kernel", "lm_scatter_kernel",
         "lm_tensor_kernel", "lm_select_kernel", "fs_scan_kernel")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else f"profiles/traffic_{cfg}.json"
    searches = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    scan_path = sys.argv[5] if len(sys.argv) > 5 else None
    nprobe = int(sys.argv[6]) if len(sys.argv) > 6 else None
    if rep.endswith(".csv"):   # ncu --csv --log-file of a metrics-only run
        txt = open(rep).read()
        lines = txt.splitlines()
        lines = lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]
        rows = list(csv.reader(lines))
        return from_long_csv(rows, cfg, out, searches, scan_path, nprobe, rep)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    it, ik = hdr.index("gpu__time_duration.sum"), hdr.index("Kernel Name")
    per = {}
    for r in rows[2:]:
        name = r[ik].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        b = (float(r[ir]) * UNIT.get(units[ir], 1) + float(r[iw]) * UNIT.get(units[iw], 1))
        per.setdefault(name, []).append((b, float(r[it])))
    kern = {k: {"dram_bytes_per_search": sum(x[0] for x in v) / searches,
                "duration_per_search": sum(x[1] for x in v) / searches,
                "duration_unit": units[it], "launches": len(v)} for k, v in per.items()}
    stage = sum(v["dram_bytes_per_search"] for k, v in kern.items() if k in STAGE)
    json.dump({"config": cfg, "source": rep, "scan_path": scan_path, "nprobe": nprobe,
               "dram_bytes_per_launch": stage,
               "stage_kernels": [k for k in kern if k in STAGE], "kernels": kern},
              open(out, "w"), indent=1)
    print(json.dumps({"dram_bytes_per_launch": stage, "kernels": list(kern)}))


def from_long_csv(rows, cfg, out, searches, scan_path, nprobe, rep):
    """ncu --metrics ... --csv (one row per (launch, metric))."""
    hdr = rows[0]
    iid, ik, im, iu, iv = (hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"),
                           hdr.index("Metric Unit"), hdr.index("Metric Value"))
    launches = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = launches.setdefault(r[iid], {"name": r[ik]})
        v = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1)
        d[r[im]] = v if r[iu] in UNIT else float(r[iv].replace(",", ""))
        d[r[im] + ".unit"] = r[iu]
    per = {}
    for d in launches.values():
        name = d["name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        per.setdefault(name, []).append((b, d.get("gpu__time_duration.sum", 0.0)))
    kern = {k: {"dram_bytes_per_search": sum(x[0] for x in v) / searches,
                "duration_per_search_ns": sum(x[1] for x in v) / searches,
                "launches": len(v)} for k, v in per.items()}
    stage = sum(v["dram_bytes_per_search"] for k, v in kern.items() if k in STAGE)
    json.dump({"config": cfg, "source": rep, "scan_path": scan_path, "nprobe": nprobe,
               "dram_bytes_per_launch": stage,
               "stage_kernels": [k for k in kern if k in STAGE], "kernels": kern},
              open(out, "w"), indent=1)
    print(json.dumps({"dram_bytes_per_launch": stage, "kernels": list(kern)}))


if __name__ == "__main__":
    main()
