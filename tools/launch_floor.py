"""Device time (CUDA events on the launch stream) of one rollout launch for
tiny batches: the launch + setup floor (E1: playouts end at the root action)
against real playouts (c3_d1), both kernels.   python tools/launch_floor.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2403_10720_b200 import dvc
    out = {}
    for name in ("tests/golden/E1.json", "fixtures/c2_d1.json", "fixtures/c3_d1.json"):
        d = json.load(open(os.path.join(ROOT, name)))
        st = dvc.encode(d)
        codes = st.legal_actions()[:1]
        hist = torch.zeros((1, st.players), dtype=torch.int64, device="cuda")
        for kern in (0, 1):
            with dvc.options(kernel=kern):
                for n in (1, 32, 1024):
                    ts = []
                    for _ in range(60):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        dvc.rollout_batch_async(st, codes, 1, 0, 0, n, hist)
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1000)
                    ts.sort()
                    out["%s k%d n%d" % (os.path.basename(name), kern, n)] = [round(ts[0], 2), round(ts[30], 2)]
    print(json.dumps(out, indent=0))


if __name__ == "__main__":
    main()
