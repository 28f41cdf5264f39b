"""Copy the outputs of scripts/final_validation.sh (gpurun_out/) into the tracked profiles/ files
of a round:

    python scripts/collect_profiles.py r02 "final validation run"

bench_final.json -> <r>_bench.json; all_*.json -> <r>_all_configs.jsonl; bench_ref.json ->
<r>_bench_reference.json; parity.jsonl -> <r>_parity.json (margins per case + the overall maximum);
launches.csv -> <r>_launches.csv + <r>_launches_summary.json; the two `ncu --set full` summaries
with their hottest SASS lines -> <r>_step_kernel_k16_ncu_full.txt, <r>_resident_torus16_ncu.txt.
"""
import json
import math
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")


def last_json(path):
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1])


def main(rnd, note):
    shutil.copy(os.path.join(GO, "bench_final.json"), os.path.join(PR, f"{rnd}_bench.json"))
    shutil.copy(os.path.join(GO, "bench_ref.json"), os.path.join(PR, f"{rnd}_bench_reference.json"))
    with open(os.path.join(PR, f"{rnd}_all_configs.jsonl"), "w") as f:
        for w in ("gmrf32", "torus256", "gmrf1000", "btb4m", "gmrf5000_dbl"):
            f.write(json.dumps(last_json(os.path.join(GO, f"all_{w}.json"))) + "\n")
    cases = [json.loads(ln) for ln in open(os.path.join(GO, "parity.jsonl")) if ln.startswith("{")]
    worst = max(c["rel_err_gamma"] for c in cases)
    parity = {
        "what": "full-m GPU parity vs the oracle's tables (tests/test_parity_full_gpu.py), every probe of "
                "BASELINE configs[0..4], bench launch configurations k=16 and k=64 (32 for torus256), "
                "Algorithm 1 and moment doubling, with the kernel schedule each case ran",
        "box": f"B200 (gpurun), {rnd}, {note}",
        "tolerances": cases[0]["tolerances"],
        "max_rel_err_gamma_overall": worst,
        "margin_orders_of_magnitude_gamma": math.log10(1e-10 / worst) if worst > 0 else None,
        "cases": cases,
    }
    json.dump(parity, open(os.path.join(PR, f"{rnd}_parity.json"), "w"), indent=1)
    shutil.copy(os.path.join(GO, "launches.csv"), os.path.join(PR, f"{rnd}_launches.csv"))
    subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "launch_summary.py"),
                           os.path.join(PR, f"{rnd}_launches.csv"), os.path.join(PR, f"{rnd}_launches_summary.json"),
                           f"ncu launch list of the headline bench command ({note})"])
    for summ, sass, dst in (("k16_summary.txt", "k16_sass.csv.gz", f"{rnd}_step_kernel_k16_ncu_full.txt"),
                            ("res16_summary.txt", "res16_sass.csv.gz", f"{rnd}_resident_torus16_ncu.txt")):
        txt = open(os.path.join(GO, summ)).read()
        hot = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sass_hot.py"), os.path.join(GO, sass), "16"],
                             capture_output=True, text=True).stdout
        open(os.path.join(PR, dst), "w").write(txt + hot)
    t = open(os.path.join(GO, "t_gpu_full.log")).read().strip().splitlines()[-1]
    print("gpu tests:", t)
    print("bench:", {k: last_json(os.path.join(GO, "bench_final.json")).get(k) for k in ("value", "ms_per_step")})
    print("parity worst rel err:", worst, "cases", len(cases))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "final validation run")
