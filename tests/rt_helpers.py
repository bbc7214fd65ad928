"""Shared test helpers (kept out of conftest so test modules can import them)."""
import importlib.util
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def _make_golden_module():
    spec = importlib.util.spec_from_file_location("rt_make_golden", os.path.join(GOLDEN, "make_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def import_reference():
    return _make_golden_module().import_reference()
