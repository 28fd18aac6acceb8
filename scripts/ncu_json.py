"""profiles/*_ncu_query_cfg3.json from `ncu --page raw --csv` exports of the query
kernels: per kernel duration, DRAM bytes (GB), instructions, IPC, occupancy.
usage: ncu_json.py OUT.json RAW.csv [RAW2.csv ...]"""
import csv, json, re, sys

SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
TSCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def label(name):
    m = re.match(r"void (k_\w+)<([^>]*)>", name)
    if not m:
        return name.split("(")[0]
    k, a = m.group(1), [x.strip() for x in m.group(2).split(",")]
    mode = {"0": "COUNT", "1": "EMIT_RETEST", "2": "EMIT"}.get(a[0], a[0])
    fmt = "" if a[1] == "0" else ",pairs"
    seq = ",seq" if len(a) >= 4 and a[3] in ("1", "true") else ""
    wide = ",wide" if len(a) >= 3 and a[2] in ("1", "true") and k == "k_query" else ""
    return f"{k}<{mode}{fmt}{wide}{seq}>"


out = {"source": "ncu --set full --clock-control none, one launch each (scripts/ncu_kq.sh; "
                 "config in the file name)", "kernels": {}}
for path in sys.argv[2:]:
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}
    for r in rows[2:]:
        g = lambda k: float(r[col[k]]) if r[col[k]] not in ("", "n/a") else None
        name = r[col["Kernel Name"]]
        out["kernels"].setdefault(label(name), {
            "name": name,
            "duration_ms": g("gpu__time_duration.sum") * TSCALE[u[col["gpu__time_duration.sum"]]],
            "dram_read_GB": g("dram__bytes_read.sum") * SCALE[u[col["dram__bytes_read.sum"]]],
            "dram_write_GB": g("dram__bytes_write.sum") * SCALE[u[col["dram__bytes_write.sum"]]],
            "inst_executed": g("smsp__inst_executed.sum"),
            "ipc": g("sm__inst_executed.avg.per_cycle_active"),
            "achieved_occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "threads_per_inst": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
            "branch_targets_uniform_pct": g("smsp__sass_average_branch_targets_threads_uniform.pct"),
            "l2_hit_pct": g("lts__t_sector_hit_rate.pct"),
            "top_stalls_per_issue": dict(sorted(
                ((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                  round(float(r[i]), 2)) for k, i in col.items()
                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
                 and r[i] not in ("", "n/a")), key=lambda kv: -kv[1])[:5])})
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps({k: (v["duration_ms"], round(v["dram_read_GB"] + v["dram_write_GB"], 3))
                  for k, v in out["kernels"].items()}))
