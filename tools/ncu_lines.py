"""Per-source-line dynamic cost of a kernel from an ncu report (thread-
instructions executed, warp-instructions, stall samples), hottest first.

    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top] [playouts]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    nplay = float(sys.argv[3]) if len(sys.argv) > 3 else 0
    f, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r) if h not in ("Source",)}
            hdr["Source"] = 1
        elif r and r[0] not in ("", "Function Name") and hdr and len(r) > 8:
            def num(k):
                v = r[hdr[k]]
                return float(v) if v not in ("-", "") else 0.0
            try:
                vals = (num("Thread Instructions Executed"), num("Instructions Executed"),
                        num("Warp Stall Sampling (All Samples)"))
            except ValueError:
                continue
            out.append(vals + ("%s:%s" % (f, r[0]), r[1].strip()[:90]))
            continue
            out.append((num("Thread Instructions Executed"), num("Instructions Executed"),
                        num("Warp Stall Sampling (All Samples)"), "%s:%s" % (f, r[0]), r[1].strip()[:90]))
    T = sum(o[0] for o in out)
    W = sum(o[1] for o in out)
    S = sum(o[2] for o in out) or 1
    print("thread-inst %.4g  warp-inst %.4g  eta %.3f" % (T, W, T / W / 32))
    for o in sorted(out, key=lambda o: -o[0])[:top]:
        per = (" %7.1f/playout" % (o[0] / nplay)) if nplay else ""
        print("%5.1f%% thr %5.1f%% stall  eta %.2f%s  %-16s %s" % (100 * o[0] / T, 100 * o[2] / S,
              o[0] / max(o[1], 1) / 32, per, o[3], o[4]))


if __name__ == "__main__":
    main()
