"""Summaries of ncu captures for profiles/ (run here, no GPU needed).

    summarize_ncu.py full <rep.ncu-rep> <out.json>        # --set full capture
    summarize_ncu.py launches <launches.csv> <out.json>    # gpu__time_duration list
    summarize_ncu.py fullcsv <out.json> <raw.csv>...       # `ncu -i rep --page raw --csv` exports (units row)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    "pipe_alu_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    "pipe_fma_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "pipe_lsu_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    "warp_insts": ("smsp__inst_executed.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "local_spill_ld_sectors": ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", 1),
    "local_spill_st_sectors": ("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "divergent_branch_targets": ("smsp__sass_branch_targets_threads_divergent.sum", 1),
    "sm_mhz": ("sm__cycles_elapsed.avg.per_second", 1e-6),
}


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")}
        for k, (m, sc) in KEYS.items():
            v = num(d.get(m))
            e[k] = None if v is None else v * sc
        stalls = {k.split("stalled_")[1]: num(v) for k, v in d.items()
                  if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and num(v)}
        tot = sum(stalls.values()) or 1
        e["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        res.append(e)
    json.dump(res, open(out, "w"), indent=1)
    for e in res:
        print(json.dumps(e)[:400])


UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
        "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "hz": 1.0, "Khz": 1e3,
        "Mhz": 1e6, "Ghz": 1e9}


def fullcsv(out, *files):
    """Same summary as full() from raw CSV exports (second row = units; values
    converted to base units: seconds, bytes, Hz)."""
    res = []
    for fn in files:
        rows = list(csv.reader(open(fn)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
            e = {"kernel": d.get("Kernel Name", "").split("(")[0], "source": fn.split("/")[-1]}
            for k, (m, sc) in KEYS.items():
                v = num(d.get(m))
                if v is not None:
                    v *= UNIT.get(u.get(m, ""), 1.0)
                    if k == "duration_ms":
                        v *= 1e3
                    elif k == "sm_mhz":
                        v *= 1e-6
                e[k] = v
            stalls = {k.split("stalled_")[1]: num(v) for k, v in d.items()
                      if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and num(v)}
            tot = sum(stalls.values()) or 1
            e["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
            res.append(e)
    json.dump(res, open(out, "w"), indent=1)
    for e in res:
        print(json.dumps(e)[:600])


def launches(fn, out):
    rows = list(csv.reader(open(fn)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[h + 1:]:
        v = num(r[vi])
        if v is None:
            continue
        u = r[ui]
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    res = [{"kernel": k, "launches": cnt[k], "total_ms": round(tot[k], 4), "mean_ms": round(tot[k] / cnt[k], 4),
            "share_pct": round(100 * tot[k] / T, 2)} for k in sorted(tot, key=lambda k: -tot[k])]
    json.dump({"note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare "
                       "shares)", "kernels": res}, open(out, "w"), indent=1)
    for e in res:
        print(e)


if __name__ == "__main__":
    {"full": full, "launches": launches, "fullcsv": fullcsv}[sys.argv[1]](*sys.argv[2:])
