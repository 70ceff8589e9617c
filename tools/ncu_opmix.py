"""Dynamic instruction mix of one kernel from an ncu report's source page:
warp-instructions executed per SASS opcode, the pipe each opcode issues to,
and each pipe's implied occupancy (fraction of instructions x issue active x
cycles per warp-instruction on that pipe as ncu normalises it: ALU 2, FMA 1
(ncu's FMA figure spans both FMA-side halves), XU 8), so the pipe
utilisation ncu reports can be checked against the mix, plus the source lines
that issue the most ALU-pipe instructions.

    python tools/ncu_opmix.py REP.ncu-rep OUT.json [issue_active_pct]
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

PIPE = {}
for op in ("LOP3", "ISETP", "SEL", "SHF", "PRMT", "PLOP3", "VIMNMX", "IMNMX", "IADD3", "LEA", "MOV", "P2R", "R2P"):
    PIPE[op] = "alu"
for op in ("IMAD", "VIADD", "IMUL"):
    PIPE[op] = "fma"
for op in ("POPC", "FLO", "BREV"):
    PIPE[op] = "xu"
CYCLES = {"alu": 2, "fma": 1, "xu": 8}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    issue = float(sys.argv[3]) / 100.0 if len(sys.argv) > 3 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    f = cur = None
    iw = None
    ops = collections.Counter()
    per_line = collections.defaultdict(collections.Counter)
    text = {}
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            iw = r.index("Instructions Executed")
            continue
        if not r or iw is None:
            continue
        if r[0]:
            cur = "%s:%s" % (f, r[0])
            text[cur] = r[1].strip()[:100]
            continue
        if len(r) <= iw or r[2] in ("...", ""):
            continue
        try:
            w = float(r[iw] or 0)
        except ValueError:
            continue
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[3])
        op = m.group(1) if m else "?"
        ops[op] += w
        per_line[cur][op] += w
    tot = sum(ops.values())
    pipes = collections.Counter()
    for op, w in ops.items():
        pipes[PIPE.get(op, "other")] += w
    res = {"report": rep, "warp_inst": tot,
           "opcodes_pct": {op: round(100 * w / tot, 2) for op, w in ops.most_common(30)},
           "pipe_inst_pct": {p: round(100 * w / tot, 2) for p, w in pipes.most_common()}}
    if issue is not None:
        res["issue_active_pct"] = 100 * issue
        res["pipe_occupancy_implied_pct"] = {p: round(100 * pipes[p] / tot * issue * c, 1) for p, c in CYCLES.items()}
    hot = sorted(per_line.items(), key=lambda kv: -sum(w for o, w in kv[1].items() if PIPE.get(o) == "alu"))
    res["top_alu_lines"] = [{"line": k, "alu_pct": round(100 * sum(w for o, w in c.items() if PIPE.get(o) == "alu") / tot, 2),
                             "all_pct": round(100 * sum(c.values()) / tot, 2), "source": text.get(k, "")}
                            for k, c in hot[:15]]
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
