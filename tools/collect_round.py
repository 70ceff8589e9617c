"""Copy a tools/round_measure.sh output set into profiles/ (tracked) with
summaries: python tools/collect_round.py TAG"""
import csv
import collections
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches_summary(src, dst, tag):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, body = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in body:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:60]
        tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
        cnt[name] += 1
    T = sum(tot.values())
    with open(dst, "w") as f:
        f.write("# %s launch list: python bench.py --steps 3 --warmup 3 --no-cpu-baseline under\n" % tag)
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised per launch)\n")
        f.write("kernel,launches,total_ms,mean_ms,share_pct\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            f.write("%s,%d,%.4f,%.4f,%.2f\n" % (k, cnt[k], tot[k], tot[k] / cnt[k], 100 * tot[k] / T))


def main():
    tag = sys.argv[1]
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles")
    for name in ("bench.jsonl", "bench_reference.jsonl", "configs.jsonl"):
        if os.path.exists(os.path.join(src, name)):
            shutil.copy(os.path.join(src, name), os.path.join(dst, "%s_%s" % (tag, name.replace("configs.jsonl", "configs_c1_c4.jsonl"))))
    for f in os.listdir(src):
        if (f.endswith(".csv") or f.endswith(".jsonl")) and f.startswith(tag):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    if os.path.exists(os.path.join(src, "launches_ncu.csv")):
        shutil.copy(os.path.join(src, "launches_ncu.csv"), os.path.join(dst, "%s_launches_ncu.csv" % tag))
        launches_summary(os.path.join(src, "launches_ncu.csv"), os.path.join(dst, "%s_launches_summary.csv" % tag),
                         tag)
    summ = os.path.join(ROOT, "tools", "summarize_profile.py")
    for rep, n, out, unit in (("refill_c2", 21000000, "refill_c2_ncu.json", True),
                              ("naive_c2", 21000000, "naive_c2_ncu.json", False),
                              ("refill_c4", 10200000, "refill_c4_ncu.json", False)):
        path = os.path.join(src, rep + ".ncu-rep")
        if os.path.exists(path):
            cmd = [sys.executable, summ, path, str(n), os.path.join(dst, "%s_%s" % (tag, out))]
            if unit:
                cmd.append("--unit")
            subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL, cwd=ROOT)
    rep = os.path.join(src, "refill_c2.ncu-rep")
    summ_json = os.path.join(dst, "%s_refill_c2_ncu.json" % tag)
    if os.path.exists(rep) and os.path.exists(summ_json):
        issue = json.load(open(summ_json))["issue_active_pct"]
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_opmix.py"), rep,
                        os.path.join(dst, "%s_refill_c2_opmix.json" % tag), str(issue)], check=True, cwd=ROOT)
    print("collected", tag)


if __name__ == "__main__":
    main()
