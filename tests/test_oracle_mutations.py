"""The closed-form pins catch plausible mistakes in the oracle's own entry
points (VERDICT r01 "Next round" #1: "a -m 'not gpu' test that goes red when
oracle_t2f_sited uses a reciprocal multiply, or when the Pr line is mis-signed
in both directions").  Each case compiles a mutated copy of
oracle/nnvisr_oracle.c into a temporary library and runs the entry-point pins
(tests/test_oracle_entry_pins.py) against it in a subprocess: they must FAIL.
The unmutated source must pass the same run (control)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "nnvisr_oracle.c")

MUTATIONS = {
    "control": [],
    # reciprocal multiplication flips BT.709 full-range yellow Cb
    "reciprocal_pb": [("double Pb = (B - Y) / (2.0 * (1.0 - kb));",
                       "double Pb = (B - Y) * (1.0 / (2.0 * (1.0 - kb)));"),
                      ("*pb = (B - Y) / (2.0 * (1.0 - kb));", "*pb = (B - Y) * (1.0 / (2.0 * (1.0 - kb)));")],
    # the same misreading of the Pr line in both directions (round trips still pass)
    "mirrored_pr": [("double Pr = (R - Y) / (2.0 * (1.0 - kr));", "double Pr = (Y - R) / (2.0 * (1.0 - kr));"),
                    ("*pr = (R - Y) / (2.0 * (1.0 - kr));", "*pr = (Y - R) / (2.0 * (1.0 - kr));"),
                    ("r = Y + 2.0 * (1.0 - kr) * Pr;", "r = Y - 2.0 * (1.0 - kr) * Pr;")],
    # a transposed pair of constants in the decode direction
    "swapped_kr_kb_f2t": [("b = Y + 2.0 * (1.0 - kb) * Pb;", "b = Y + 2.0 * (1.0 - kr) * Pb;")],
    # a dropped term in G' (t2f luma)
    "dropped_kb_term": [("double Y = G + kr * (R - G) + kb * (B - G);\n                store_sample",
                         "double Y = G + kr * (R - G);\n                store_sample")],
}


@pytest.mark.parametrize("name", list(MUTATIONS))
def test_pins_catch_mutation(name, tmp_path):
    src = open(SRC).read()
    for old, new in MUTATIONS[name]:
        assert src.count(old) >= 1, (name, old)
        src = src.replace(old, new)
    c = tmp_path / "mut.c"
    so = tmp_path / "libmut.so"
    c.write_text(src)
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                           "-o", str(so), str(c), "-lm"])
    env = dict(os.environ, NNVISR_ORACLE_MUTANT_LIB=str(so))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle_entry_pins.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    if name == "control":
        assert r.returncode == 0, r.stdout[-2000:]
    else:
        assert r.returncode != 0, f"mutation {name} escaped the entry-point pins"
