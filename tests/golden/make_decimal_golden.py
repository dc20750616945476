"""tests/golden/decimal.json: DoubleWord/TripleWord.decimal_str from the REAL
reference (multiword.py:48-51, 71-75 -> ExactValue.decimal_str).  Build container only."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import HERE, _import_reference, hx  # noqa: E402


def main():
    _, _, mw, _, _ = _import_reference()
    rng = np.random.default_rng(7)
    cases = []
    for t in range(60):
        w0 = float(rng.standard_normal() * 10.0 ** int(rng.integers(-40, 40)))
        if t % 10 == 0:
            w0 = [0.0, 1.0, -9.999999999999999, 0.5, 5e-324, 1e308][t // 10]
        w1 = float(np.spacing(w0) * rng.uniform(-0.5, 0.5))
        w2 = float(np.spacing(w1) * rng.uniform(-0.5, 0.5)) if w1 else 0.0
        d = int(rng.integers(1, 70))
        cases.append({"dw": [hx(w0), hx(w1)], "tw": [hx(w0), hx(w1), hx(w2)], "digits": d,
                      "dw_str": mw.DoubleWord(w0, w1).decimal_str(d),
                      "tw_str": mw.TripleWord(w0, w1, w2).decimal_str(d),
                      "dw_default": mw.DoubleWord(w0, w1).decimal_str(),
                      "tw_default": mw.TripleWord(w0, w1, w2).decimal_str()})
    with open(os.path.join(HERE, "decimal.json"), "w") as f:
        json.dump({"cases": cases}, f, indent=0)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
