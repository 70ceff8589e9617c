"""Static per-source-line pipe mix of one kernel's SASS (no GPU):
    python tools/sass_lines.py LIB.so KERNEL_MANGLED [lo_addr hi_addr]
Instructions in [lo, hi) (hex byte offsets, default: all) are attributed to
the innermost source line nvdisasm -g reports and classed by pipe (B300
guide: IMAD* on fma; IADD3/LOP3/SHF/PRMT/ISETP/SEL/... on alu; POPC/FLO/BREV on xu)."""
import collections, os, re, subprocess, sys, tempfile

lib, fn = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.startswith("kernels") or f.endswith(".cubin")]
txt = ""
for c in cub:
    t = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, c)], capture_output=True, text=True).stdout
    if fn in t:
        txt = t
        break
sec = txt[txt.index(".text." + fn + ","):]
sec = sec[:sec.index("//---------------------", 10)] if "//---------------------" in sec[10:] else sec
ALU = {"LOP3", "SHF", "ISETP", "SEL", "IADD3", "PLOP3", "PRMT", "LEA", "VIMNMX", "SGXT", "IABS", "LOP", "P2R", "R2P",
       "IADD", "VIADDMNMX", "IMNMX", "BMSK", "MOV", "ICMP"}
XU = {"POPC", "FLO", "BREV", "MUFU"}
line = "?"
per = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for l in sec.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = "%s:%s" % (os.path.basename(m.group(1)), m.group(2))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", l)
    if not m:
        continue
    addr = int(m.group(1), 16)
    if not (lo <= addr < hi):
        continue
    op = m.group(2)
    pipe = "fma" if op.startswith("IMAD") or op in ("IMUL", "FFMA") else "alu" if op in ALU else \
        "xu" if op in XU else "viadd" if op == "VIADD" else "other"
    per[line][pipe] += 1
    tot[pipe] += 1
print("total", sum(tot.values()), dict(tot))
for k, c in sorted(per.items(), key=lambda kv: -sum(kv[1].values())):
    print("%-22s %3d  %s" % (k, sum(c.values()), dict(c)))
