"""Summarise an `ncu --page source --csv` SASS listing: hottest instructions by
warp-stall samples, with executed counts and average active threads.

    ncu -i prof.ncu-rep --page source --csv > src.csv; python tools/ncu_sass.py src.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    S = ix["Warp Stall Sampling (All Samples)"]
    E = ix["Instructions Executed"]
    T = ix["Avg. Threads Executed"]
    tot = sum(float(r[S] or 0) for r in body)
    texec = sum(float(r[E] or 0) for r in body)
    print("instructions:", len(body), "samples:", tot, "warp-inst executed:", texec)
    if "--list" in sys.argv:
        for n, r in enumerate(body):
            print("%4d %6s %12s %5s  %s" % (n, r[S], r[E], r[T], r[ix["Source"]].strip()))
        return
    order = sorted(range(len(body)), key=lambda i: -float(body[i][S] or 0))
    for i in order[:top]:
        r = body[i]
        print("%4d %6s (%4.1f%%) exec=%10s thr=%5s  %s" % (i, r[S], 100 * float(r[S] or 0) / tot, r[E], r[T],
                                                          r[ix["Source"]].strip()))


if __name__ == "__main__":
    main()
