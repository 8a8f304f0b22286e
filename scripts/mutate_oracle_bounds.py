#!/usr/bin/env python
"""Mutation test of the oracle's run-time gap bound.

For every additive term of the local error bounds (eg, es, el, ez, eq, eu, ey, ex,
er, ek, ew) and of the bound recursions (Dz_i, Ds_i, Dw_1, f_1) in
oracle/oracle.c's automated-replacement code, and for every numeric coefficient
(2.0 <-> 3.0, 4.0 -> 3.0), build a mutant oracle, run
tests/test_oracle_autorr.py + tests/test_oracle_autorr_terms.py against it and
record whether the mutant is caught.  Restores oracle.c afterwards.

    python scripts/mutate_oracle_bounds.py      # ~2 min
"""
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")
TARGETS = ["eg", "es", "el", "ez", "eq", "eu", "ey", "ex", "er", "ek", "ew",
           "Dz_i", "Ds_i", "Dw_1", "f_1"]


def split_terms(rhs):
    """top-level '+' terms of an expression"""
    out, depth, cur = [], 0, ""
    for ch in rhs:
        depth += ch == "("
        depth -= ch == ")"
        if ch == "+" and depth == 0:
            out.append(cur)
            cur = ""
        else:
            cur += ch
    out.append(cur)
    return out


def mutants(text):
    lines = text.split("\n")
    # the automated-replacement block of orc_pbicgstab: statements start with
    # "const double <name> =" or "<name> =" and may span lines until ';'
    start = text.index("/* eq:errbounds1-4 without the common factor eps */")
    stop = text.index("/* lines 17-20 (P:183-186) */")
    block = text[start:stop]
    for name in TARGETS:
        m = re.search(r"(?:const double )?\b" + re.escape(name) + r" = ([^;]*);", block)
        if not m:
            raise SystemExit(f"statement {name} not found")
        rhs = m.group(1)
        terms = split_terms(rhs)
        for k in range(len(terms)):
            if len(terms) == 1:
                break
            new = "+".join(t for j, t in enumerate(terms) if j != k)
            yield f"{name}: drop term {k} ({terms[k].strip()})", \
                text[:start] + block.replace(m.group(0), m.group(0).replace(rhs, new), 1) + text[stop:]
        for coef, repl in (("2.0", "3.0"), ("3.0", "2.0"), ("4.0", "3.0")):
            for occ in [mm.start() for mm in re.finditer(re.escape(coef), rhs)]:
                new = rhs[:occ] + repl + rhs[occ + len(coef):]
                yield f"{name}: {coef} -> {repl} at {occ}", \
                    text[:start] + block.replace(m.group(0), m.group(0).replace(rhs, new), 1) + text[stop:]


def main():
    orig = open(SRC).read()
    backup = SRC + ".bak"
    shutil.copy(SRC, backup)
    results = []
    try:
        for desc, mut in mutants(orig):
            with open(SRC, "w") as f:
                f.write(mut)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x",
                                "tests/test_oracle_autorr.py", "tests/test_oracle_autorr_terms.py"],
                               cwd=ROOT, capture_output=True, text=True)
            caught = r.returncode != 0
            results.append((desc, caught))
            print(("CAUGHT  " if caught else "MISSED  ") + desc, flush=True)
    finally:
        shutil.copy(backup, SRC)
        os.remove(backup)
        subprocess.run([sys.executable, "-c", "from oracle import oracle as o; o.build(force=True)"],
                       cwd=ROOT)
    n = len(results)
    c = sum(1 for _, k in results if k)
    print(f"{c} / {n} mutants caught")
    return 0 if c == n else 1


if __name__ == "__main__":
    sys.exit(main())
