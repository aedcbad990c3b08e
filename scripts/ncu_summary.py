"""Dev tool: regenerate profiles/r01_ncu_full_summary.json and
profiles/ncu_gather_summary.json (read by bench.py as roofline.traffic) from
an `ncu --set full` report of one gather_kernel launch:
    python scripts/ncu_summary.py gpurun_out/final/prof_gather.ncu-rep"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    names, units, vals = rows[0], rows[1], rows[2]
    old = json.load(open(os.path.join(ROOT, "profiles", "r01_ncu_full_summary.json")))
    keep = list(old["metrics"].keys())
    metrics = {}
    for k in keep:
        if k in names:
            i = names.index(k)
            metrics[k] = [vals[i], units[i]]
    g = lambda k: float(vals[names.index(k)].replace(",", ""))   # noqa: E731
    st_req = g("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum")
    st_sec = g("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum")
    kname = vals[names.index("Kernel Name")] if "Kernel Name" in names else old["kernel"]
    out = {"kernel": kname, "source": old["source"], "metrics": metrics,
           "derived": {"global_store_sectors_per_request": round(st_sec / st_req, 3),
                       "warp_efficiency_threads_per_inst":
                           vals[names.index("smsp__thread_inst_executed_per_inst_executed.ratio")]}}
    json.dump(out, open(os.path.join(ROOT, "profiles", "r01_ncu_full_summary.json"), "w"), indent=1)
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
    rd = g("dram__bytes_read.sum") * scale[units[names.index("dram__bytes_read.sum")]]
    wr = g("dram__bytes_write.sum") * scale[units[names.index("dram__bytes_write.sum")]]
    dur = f'{vals[names.index("gpu__time_duration.sum")]} {units[names.index("gpu__time_duration.sum")]}'
    summ = {"config": "c2_1080p_sparse", "fmt": "f32", "src": "rgb24", "kernel": "void gather_kernel<0, 0>",
            "dram_bytes_per_step": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr, "ncu_duration": dur,
            "source": "ncu --set full --clock-control none, one launch (bench.py --depth 1); "
                      "profiles/r01_ncu_full_summary.json"}
    json.dump(summ, open(os.path.join(ROOT, "profiles", "ncu_gather_summary.json"), "w"), indent=1)
    print(json.dumps(summ))


if __name__ == "__main__":
    main(sys.argv[1])
