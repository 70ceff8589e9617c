"""Where lanes are lost: per source line, warp-instructions x 32 minus
thread-instructions (the SIMT-efficiency loss), largest first.

    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_loss.py src.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    f = hdr = None
    out = []
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r) if h != "Source"}
        elif r and r[0] not in ("", "Function Name") and hdr and len(r) > 8:
            try:
                t = float(r[hdr["Thread Instructions Executed"]] or 0)
                w = float(r[hdr["Instructions Executed"]] or 0)
            except ValueError:
                continue
            out.append((32 * w - t, t, w, "%s:%s" % (f, r[0]), r[1].strip()[:80]))
    lost = sum(o[0] for o in out)
    T = sum(o[1] for o in out)
    W = sum(o[2] for o in out)
    print("warp-inst %.4g  thread-inst %.4g  lost lane-slots %.3g  eta %.3f" % (W, T, lost, T / (lost + T)))
    for o in sorted(out, key=lambda o: -o[0])[:top]:
        print("%5.1f%% of loss  %5.2f%% of warp-inst  eta %.2f  %-18s %s" % (
            100 * o[0] / lost, 100 * o[2] / W, o[1] / o[2] / 32 if o[2] else 0, o[3], o[4]))


if __name__ == "__main__":
    main()
