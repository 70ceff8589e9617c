"""kernel option 3 (refill2, two playouts per lane) against kernel 0 (refill,
oracle-parity-tested): identical histograms on every fixture, plain, CRN and
through the flat search; prints one JSON line."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2403_10720_b200 import dvc
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
    bad = []
    for path in sorted(glob.glob(os.path.join(ROOT, "fixtures", "*.json"))):
        st = dvc.encode(json.load(open(path)))
        codes = st.legal_actions()
        res = {}
        for k in (0, 3):
            with dvc.options(kernel=k):
                res[k] = (dvc.rollout_batch_ex(st, codes, 5, 3, 17, 17 + n).tolist(),
                          dvc.rollout_batch_ex(st, codes, 6, 0, 0, n // 3, crn=True).tolist(),
                          dvc.mcts_search(st, 16, 2048, 7, flat=1))
        if res[0] != res[3]:
            bad.append(os.path.basename(path))
    print(json.dumps({"fixtures": len(glob.glob(os.path.join(ROOT, "fixtures", "*.json"))), "mismatch": bad}))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
