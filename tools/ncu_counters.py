"""Per-launch counters of one ncu --set full capture -> profiles/ncu_traffic.json (read by bench.py's
roofline).  python tools/ncu_counters.py REPORT.ncu-rep KEY [kernel-regex] [committed-summary]
(KEY e.g. cfg4-k4; the summary path, under profiles/, is recorded as the evidence)"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def read(rep, kregex=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if kregex and not re.search(kregex, name):
            continue
        def get(metric, unit_to=None):
            i = hdr.index(metric)
            v = float(r[i].replace(",", ""))
            return v * SCALE.get(units[i], 1.0) if unit_to else v
        def opt(metric, unit_to=None):
            try:
                return get(metric, unit_to)
            except (ValueError, IndexError):
                return 0.0
        red = get("lts__t_requests_srcunit_tex_op_red.sum")
        atom = opt("lts__t_requests_srcunit_tex_op_atom_dot_alu.sum") + opt("lts__t_requests_srcunit_tex_op_atom_dot_cas.sum")
        hit = opt("lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum")
        miss = opt("lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum")
        return {
            "kernel": name[:120],
            "duration_ms": get("gpu__time_duration.sum", "ms"),
            "dram_bytes": get("dram__bytes_read.sum", "b") + get("dram__bytes_write.sum", "b"),
            "l2_red_requests": red,
            "l2_atom_requests": atom,
            "l2_red_sectors": opt("lts__t_sectors_srcunit_tex_op_red.sum"),
            "l2_red_hit_pct": 100.0 * hit / max(hit + miss, 1.0),
            "l2_red_unit_pct": opt("lts__t_sectors_srcunit_tex_op_red.avg.pct_of_peak_sustained_elapsed"),
            "l2_hit_pct": opt("lts__t_sector_hit_rate.pct"),
            "issue_frac": opt("sm__inst_executed.avg.pct_of_peak_sustained_elapsed") / 100.0,
            "warps_active_pct": opt("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "warp_insts": opt("smsp__inst_executed.sum"),
        }
    raise SystemExit(f"no kernel matching {kregex} in {rep}")


def main():
    rep, key = sys.argv[1], sys.argv[2]
    kregex = sys.argv[3] if len(sys.argv) > 3 else "k_enum"
    c = read(rep, kregex)
    c["report"] = sys.argv[4] if len(sys.argv) > 4 else os.path.relpath(rep, ROOT)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = {}
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
    d["_source"] = ("ncu --set full --clock-control none, one launch (tools/profile_enum.py); "
                    "tools/ncu_counters.py; per launch")
    d[key] = c
    with open(path, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    print(json.dumps({key: c}, indent=1))


if __name__ == "__main__":
    main()
