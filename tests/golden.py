"""Parser for tests/golden/*.txt fixtures (name | kind | inputs | expected | citation)."""
import ast
import math
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _val(s):
    s = s.strip()
    if s in ("inf", "+inf"):
        return math.inf
    if s == "-inf":
        return -math.inf
    return ast.literal_eval(s)


def load(fname="spec_examples.txt"):
    rows = {}
    with open(os.path.join(HERE, fname)) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            name, kind, inputs, expected, cite = [c.strip() for c in line.split("|", 4)]
            kv = {}
            for tok in inputs.replace(" p=", " ;p=").replace(" C=", " ;C=").replace(" C0=", " ;C0=").split(";"):
                tok = tok.strip()
                if not tok:
                    continue
                for part in ([tok] if tok.startswith(("A=", "C=", "C0=")) else tok.split()):
                    k, v = part.split("=", 1)
                    kv[k] = v
            rows[name] = dict(kind=kind, inputs=kv, expected=_val(expected), cite=cite)
    return rows


def matrix(s):
    s = s.strip()
    if s.startswith("diag("):
        return np.diag([float(x) for x in s[5:-1].split(",")])
    return np.array(ast.literal_eval(s), dtype=np.float64)
