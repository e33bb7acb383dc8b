"""Golden fixtures for the text format, from the REFERENCE's polytext module
(build container only):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_polytext.py

* polytext_c1.txt: `format_system` of the C1 target system (polytext.py:154-157).
* polytext_cases.json: inputs written for this test (not taken from the
  reference's tests) with the reference parser's verdict: the parsed terms
  (exponents, coefficient as [re, im] with exact float repr) or "error".
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import nidpipe.polytext as rpt  # noqa: E402

from make_golden import ref_sys  # noqa: E402
from paper_1804_03807_b200 import configs  # noqa: E402

CASES = [
    "2 2\nx1^2 - 1;\nx1*x2 + (0.5-0.25*i)*x2^3 - 2.5e-1;",
    "3 1\n(1.0+2.0*i)*x1*x3^2*x1 - -x2 + 3*2*x2;",
    "1 1\n.5*x1 + 1.e2 - 7;",
    "2 1\n(1e-3+1E+2*i)*x2^10 + x1 * x2 * 2;",
    "2 2\n- x1 + x2;\n+ (0.0-1.0*i);",
    "2 1\n(1.5)*x1 + (2i) + (-0.25*i)*x2;",
    "2 1\nx1^2*x1^3 - 4*-2*x2;",
    "1 0\n",
    "2 1\n(0.1+0.2*i)*x1 + (0.1-0.2*i)*x1 + 0*x2;",
    # errors
    "2 1\nx3 + 1;",
    "2 1\ny1 + 1;",
    "2 2\nx1 + 1;",
    "2 1\nx1 + (1+2*i;",
    "2 1\n2x1 + 1;",
    "2 1\nx1^-2 + 1;",
    "2 1\nx1 ** x2;",
    "2\nx1;",
    "",
    "a b\nx1;",
    "2 1\nx1 + (1+*i);",
    "0 0\n",
]


def main():
    c1 = configs.c1()
    with open(os.path.join(HERE, "polytext_c1.txt"), "w", encoding="utf-8") as fh:
        fh.write(rpt.format_system(ref_sys(c1.target)))
    out = []
    for text in CASES:
        try:
            f = rpt.parse_system(text)
            polys = [[[list(e), [repr(c.real), repr(c.imag)]] for e, c in p.terms] for p in f.polys]
            out.append({"text": text, "nvars": f.nvars, "polys": polys, "formatted": rpt.format_system(f)})
        except rpt.ParseError:
            out.append({"text": text, "error": True})
    with open(os.path.join(HERE, "polytext_cases.json"), "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1)
    print(sum(1 for o in out if "error" in o), "errors of", len(out))


if __name__ == "__main__":
    main()
