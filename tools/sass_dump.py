"""Print the SASS of one kernel of libdvc.so (static, no GPU).
    python tools/sass_dump.py [kernel-substring] [from-line] [to-line]"""
import re
import subprocess
import sys

name = sys.argv[1] if len(sys.argv) > 1 else "rollout_refill_kernelILi2ELb0ELb1E"
a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = int(sys.argv[3]) if len(sys.argv) > 3 else 10 ** 9
out = subprocess.run(["cuobjdump", "-sass", "paper_2403_10720_b200/libdvc.so"], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", out):
    if name in f.split("\n")[0]:
        lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", l).strip() for l in f.split("\n") if re.search(r"/\*[0-9a-f]{4}\*/", l)]
        for i, l in enumerate(lines):
            if a <= i <= b:
                print(i, l)
        break
