"""Opcode mix of one kernel in libdvc.so (static SASS, no GPU needed).

    python tools/sass_mix.py [kernel-substring]   (default: refill kernel <2, false, true>)
"""
import collections
import re
import subprocess
import sys

name = sys.argv[1] if len(sys.argv) > 1 else "rollout_refill_kernelILi2ELb0ELb1E"
out = subprocess.run(["cuobjdump", "-sass", "paper_2403_10720_b200/libdvc.so"], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    if name in f.split("\n")[0]:
        ops = re.findall(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", f)
        c = collections.Counter(o for o in ops)
        alu = sum(v for k, v in c.items() if k in ("LOP3", "SHF", "ISETP", "SEL", "VIADD", "IADD3", "PLOP3", "P2R", "R2P",
                                                    "PRMT", "LEA", "VIMNMX", "VIADDMNMX", "SGXT", "IABS", "LOP", "SHL", "SHR"))
        xu = sum(v for k, v in c.items() if k in ("POPC", "FLO", "BREV", "MUFU", "I2F", "F2I"))
        fma = sum(v for k, v in c.items() if k.startswith("IMAD") or k in ("IMUL", "FFMA"))
        print(f.split("\n")[0][:100])
        print("total", sum(c.values()), "alu", alu, "xu", xu, "fma", fma)
        print(c.most_common(25))
        break
