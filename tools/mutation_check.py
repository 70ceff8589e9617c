"""Mutation check of the oracle pins (VERDICT r01 "Next round" 1): copy the
repo's tests + oracle to a scratch dir, apply one textual mutation to
oracle/game.py, run the oracle pin tests there, and report whether they fail.

    python tools/mutation_check.py            # all mutations
"""
import os, shutil, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    # next_mover does not skip eliminated seats (SPEC:186 broken)
    "next_mover_no_skip": (
        "        for d in range(1, P + 1):\n            p = (self.g + d) % P\n            if self.alive(p):\n                return p\n",
        "        return (self.g + 1) % P\n"),
    # a numbered key goes LEFT of a joker in its gap (SPEC:107 broken)
    "insert_left_of_joker": (
        "            if not self.rules.is_joker(k) and k > t:\n                i = idx\n                break\n",
        "            if not self.rules.is_joker(k) and k > t:\n                i = idx\n                break\n"
        "        while i > 0 and self.rules.is_joker(ln[i - 1][0]):\n            i -= 1\n"),
    # empty pool: a wrong guess reveals the RIGHTMOST hidden tile (SPEC:184 broken)
    "rightmost_hidden": (
        "        for idx, (_, r) in enumerate(self.lines[p]):\n            if not r:\n                return idx\n",
        "        for idx in range(len(self.lines[p]) - 1, -1, -1):\n            if not self.lines[p][idx][1]:\n                return idx\n"),
}

TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_rules.py"]


def run(name, old, new):
    tmp = tempfile.mkdtemp(prefix="mut_")
    for sub in ("oracle", "tests", "fixtures"):
        shutil.copytree(os.path.join(ROOT, sub), os.path.join(tmp, sub))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
    p = os.path.join(tmp, "oracle", "game.py")
    s = open(p).read()
    assert s.count(old) == 1, name
    open(p, "w").write(s.replace(old, new))
    r = subprocess.run([sys.executable, "-m", "pytest", *TESTS, "-q", "-p", "no:cacheprovider",
                        "-k", "not python_oracle_equals_cpp"], cwd=tmp, capture_output=True, text=True)
    shutil.rmtree(tmp, ignore_errors=True)
    last = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
    return r.returncode, last


if __name__ == "__main__":
    for name, (old, new) in MUTATIONS.items():
        rc, last = run(name, old, new)
        print("%-22s %s  (%s)" % (name, "CAUGHT" if rc != 0 else "MISSED", last))
