"""Parsers for the hand-worked fixtures in tests/golden/ (test helper only)."""
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DBL_MIN = 2.2250738585072014e-308


def parse_value(tok: str) -> float:
    if tok.startswith("prev(") and tok.endswith(")"):
        return math.nextafter(parse_value(tok[5:-1]), 0.0)
    if tok == "DBL_MIN":
        return DBL_MIN
    if tok == "MAXSUB":
        return math.nextafter(DBL_MIN, 0.0)
    return float(tok)  # handles inf, -inf, nan, -0.0


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip()
            if line:
                yield line.split()


def lower_bound_cases():
    """{table_name: (X, [(y, expected), ...])}"""
    tables = {}
    for tok in _lines("lower_bound_cases.txt"):
        if tok[0] == "table":
            tables[tok[1]] = (np.array([parse_value(t) for t in tok[2:]]), [])
        elif tok[0] == "case":
            tables[tok[1]][1].append((parse_value(tok[2]), int(tok[3])))
    return tables


def interp_cases():
    grid, cases = {}, []
    for tok in _lines("interp2d_cases.txt"):
        if tok[0] == "grid":
            grid[tok[1]] = np.array([parse_value(t) for t in tok[2:]])
        elif tok[0] == "case":
            cases.append(tuple(parse_value(t) for t in tok[1:4]) + (int(tok[4]), int(tok[5])))
    R, T = grid["R"], grid["T"]
    G = grid["G"].reshape(R.size, T.size)
    return R, T, G, cases
