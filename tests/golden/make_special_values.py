"""Writes tests/golden/special_values.csv with mpmath (independent of oracle/ and of the CUDA path)."""
import mpmath as mp

mp.mp.dps = 40
rows = [("E1", 1.0, None, mp.e1(1)), ("E1", 0.01, None, mp.e1(0.01)), ("E1", 10.0, None, mp.e1(10)),
        ("erfc", 1.0, None, mp.erfc(1)), ("k0", 1.0, None, mp.besselk(0, 1))]
for a, b in [(1.0, 1.0), (40.0, 0.01), (0.001, 0.0001), (9.87, 2.0), (0.2, 30.0)]:
    rows.append(("K0inc", a, b, mp.quad(lambda t: mp.exp(-mp.mpf(a) / t - mp.mpf(b) * t) / t,
                                        [0, 1e-5, 1e-4, 1e-3, 0.01, 0.05, 0.1, 0.25, 0.5, 1])))
with open(__file__.replace("make_special_values.py", "special_values.csv"), "w") as f:
    f.write("# Special-function values computed with mpmath (dps=40) by tests/golden/make_special_values.py;\n")
    f.write("# independent of this repo's code.  E1(1) also appears in SPEC.md S:115, erfc(1) in S:89.\n")
    f.write("# K0inc(a,b) = int_0^1 exp(-a/t - b t) dt/t, the definition at PAPER.md P:95.\n")
    f.write("# name,arg1,arg2,value\n")
    for n, a, b, v in rows:
        f.write(f"{n},{a},{'' if b is None else b},{mp.nstr(v, 30)}\n")
