"""Parse tests/golden/*.txt fixtures (test infrastructure)."""
from __future__ import annotations

import os
import re

import dm_inputs as g

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def graph_from_name(name: str):
    name = name.strip()
    m = re.fullmatch(r"K(\d+)", name)
    if m:
        return g.clique(int(m.group(1)))
    m = re.fullmatch(r"C(\d+)", name)
    if m:
        return g.ring(int(m.group(1)))
    m = re.fullmatch(r"P(\d+)", name)
    if m:
        return g.path(int(m.group(1)))
    m = re.fullmatch(r"grid(\d+)x(\d+)", name)
    if m:
        return g.square_grid(int(m.group(1)), int(m.group(2)))
    m = re.fullmatch(r"star(\d+)", name)
    if m:
        return g.star(int(m.group(1)))
    raise ValueError(name)


def spec_examples():
    out = []
    with open(os.path.join(GOLDEN, "spec_examples.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, data, pat, mode, exp, cite = [x.strip() for x in line.split("|", 5)]
            out.append((name, data, pat, mode, int(exp), cite))
    return out
