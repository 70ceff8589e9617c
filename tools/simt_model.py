"""N3: the lockstep SIMT model's prediction of the naive
(thread-per-playout) kernel's warp efficiency from the oracle's playout
lengths alone (oracle/simt.py), written as an artifact beside
ncu's measured value.

    python tools/simt_model.py [--sims 2048] [--out profiles/r02_simt_model.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sims", type=int, default=2048)
    ap.add_argument("--workload", default="fixtures/c2_d1.json")
    ap.add_argument("--ncu", default="profiles/r01_naive_c2_ncu.json")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_simt_model.json"))
    args = ap.parse_args()
    import oracle
    from oracle.simt import naive_kernel_efficiency
    d = json.load(open(os.path.join(ROOT, args.workload)))
    codes = oracle.legal(d)
    eta_model = naive_kernel_efficiency(d, codes, 1, args.sims)
    res = {"workload": args.workload, "actions": len(codes), "sims_per_action": args.sims, "seed": 1,
           "eta_simt_model": eta_model,
           "model": "oracle/simt.py naive_kernel_efficiency: 32 consecutive sims of one action per warp in "
                    "lockstep, iterations = 1 start + decision steps (oracle playout lengths)",
           "command": "python tools/simt_model.py --sims %d" % args.sims}
    try:
        m = json.load(open(os.path.join(ROOT, args.ncu)))
        res["eta_simt_ncu_naive"] = m["eta_simt"]
        res["ncu_source"] = args.ncu
        res["model_minus_measured"] = eta_model - m["eta_simt"]
    except Exception:
        pass
    json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
