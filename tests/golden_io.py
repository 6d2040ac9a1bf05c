"""Loader for the committed golden fixtures (tests/golden/, generated from
the reference package by tests/golden/make_golden.py)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Case:
    def __init__(self, rec, arr):
        self.__dict__.update(rec)
        k = rec["key"]
        self.coords = tuple(arr[f"{k}_in{j}"] for j in range(rec["dim"]))
        self.verts = arr[f"{k}_verts"] if f"{k}_verts" in arr else None
        self.cand = arr[f"{k}_cand"] if f"{k}_cand" in arr else None
        self.keep = arr[f"{k}_keep"] if f"{k}_keep" in arr else None
        self.error = rec.get("error")

    def rows(self):
        return np.column_stack(self.coords)


def load():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        idx = json.load(f)
    arr = dict(np.load(os.path.join(GOLDEN, "golden.npz")))
    return [Case(r, arr) for r in idx["cases"]]


def rows_of(coords, idx):
    return np.column_stack([np.asarray(c)[idx] for c in coords]) if len(idx) else \
        np.empty((0, len(coords)))
