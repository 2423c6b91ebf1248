"""Copy one GPU run's outputs (tools/exp/final_r2.sh -> gpurun_out/) into profiles/<tag>_*
and refresh profiles/ncu_summary.json (the bench's roofline.traffic source).

    python tools/refresh_profiles.py r02a
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
WANT = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "lts__t_sectors_op_write.sum", "lts__t_requests_op_write.sum",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_metrics(rep):
    csv_path = rep.replace(".ncu-rep", "_raw.csv")
    if not os.path.exists(rep) and os.path.exists(csv_path):  # exported on the GPU box (64 MiB pull limit)
        raw = open(csv_path).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2]


def main(tag):
    for src, dst in (("bench_default.json", "bench_default.json"), ("bench_ref.json", "bench_reference.json"),
                     ("launches_c3.csv", "c3_launches.csv"), ("sweep.txt", "table1_sweep.txt"),
                     ("sustained.txt", "sustained.txt"), ("phases_c3.txt", "phases_c3.txt"),
                     ("phases_c2.txt", "phases_c2.txt"), ("gpu_tests_all.txt", "gpu_tests.txt"),
                     ("smoke.txt", "smoke.txt")):
        if os.path.exists(os.path.join(OUT, src)):
            shutil.copy(os.path.join(OUT, src), os.path.join(PROF, f"{tag}_{dst}"))
    summary_path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    for c in ("c2", "c3", "c4", "c5"):
        rep = os.path.join(OUT, f"prof_{c}.ncu-rep")
        if not os.path.exists(rep) and not os.path.exists(rep.replace(".ncu-rep", "_raw.csv")):
            continue
        h, u, v = ncu_metrics(rep)
        d = {n: (un, val) for n, un, val in zip(h, u, v)}
        lines = [f"# ncu --set full --clock-control none -k regex:fmha_fwd -s 3 -c 1 python bench.py --config {c} "
                 f"--steps 2 --warmup 3   ({tag})", f"# kernel: {d.get('Kernel Name', ('', ''))[1]}"]
        lines += [f"{w:80s} {d[w][1]:>18s} {d[w][0]}" for w in WANT if w in d]
        open(os.path.join(PROF, f"{tag}_{c}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
        rd = float(d["dram__bytes_read.sum"][1].replace(",", "")) * SCALE[d["dram__bytes_read.sum"][0]]
        wr = float(d["dram__bytes_write.sum"][1].replace(",", "")) * SCALE[d["dram__bytes_write.sum"][0]]
        summary[c] = {"dram_bytes_per_launch": int(rd + wr), "source": f"profiles/{tag}_{c}_ncu_full.txt",
                      "tensor_pipe_active_pct": float(
                          d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"][1]),
                      "kernel": d.get("Kernel Name", ("", ""))[1]}
    if "c3" in summary:
        summary["c3"]["launch_list"] = f"profiles/{tag}_c3_launches.csv"
    json.dump(summary, open(summary_path, "w"), indent=1)
    print("profiles refreshed:", tag)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "latest")
