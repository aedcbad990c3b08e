"""Dev tool: summarise one `ncu --set full` report (one kernel launch) into a
small JSON under profiles/: duration, DRAM bytes, SM issue/occupancy, pipe and
L1 utilisation, warp-stall breakdown per issue, launch resources, and the SASS
instruction mix (from the source page).

    python scripts/ncu_brief.py gpurun_out/f1/prof_gather_u8.ncu-rep profiles/r02_ncu_gather_u8_c2.json \
        --note "c2 u8, bench.py --depth 1"
"""
import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__warps_active.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "launch__waves_per_multiprocessor",
]


def ncu_csv(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu_csv(a.rep, "--page", "raw"))))
    names, units, vals = rows[0], rows[1], rows[2]
    d = {k: (vals[i], units[i]) for i, k in enumerate(names)}
    metrics = {k: " ".join(x for x in d[k] if x) for k in KEYS if k in d}
    stalls = {}
    for k, (v, _) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v:
            stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(float(v), 3)
    stalls = dict(sorted(stalls.items(), key=lambda x: -x[1]))
    # SASS instruction mix (warp-level instructions executed, by opcode)
    src = list(csv.reader(io.StringIO(ncu_csv(a.rep, "--page", "source", "--print-source", "sass"))))
    mix, tot = collections.Counter(), 0
    if len(src) > 2:
        hdr = src[1]
        i_s, i_e = hdr.index("Source"), hdr.index("Instructions Executed")
        for r in src[2:]:
            try:
                n = int(r[i_e])
            except (ValueError, IndexError):
                continue
            toks = r[i_s].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            mix[op.split(".")[0]] += n
            tot += n
    out = {"kernel": d.get("Kernel Name", ("?",))[0], "report": a.rep, "note": a.note,
           "metrics": metrics, "stalls_per_issue": stalls,
           "warp_instructions": tot,
           "instruction_mix_pct": {k: round(100.0 * v / tot, 1) for k, v in mix.most_common(16)} if tot else {}}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({"kernel": out["kernel"][:60], "duration": metrics.get("gpu__time_duration.sum"),
                      "top_stalls": list(stalls.items())[:4]}))


if __name__ == "__main__":
    main()
