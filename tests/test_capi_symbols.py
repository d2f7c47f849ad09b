"""The C-ABI library builds, loads without a GPU and exports every declared symbol."""

import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "evsim_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(evs_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_entry_points():
    names = declared_functions()
    for n in ("evs_step", "evs_step_workspace_bytes", "evs_canonical_sort", "evs_seed_pcg64"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2602_15018_b200 import _lib

    L = _lib.load()  # builds in-tree with nvcc if missing
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert L.evs_version() >= 1
    assert L.evs_error_string(1) == b"invalid argument"


def test_workspace_sizing_is_host_only():
    from paper_2602_15018_b200 import _lib

    L = _lib.load()
    p = _lib.StepParams(streams=1, frames=1, height=720, width=1280, log_eps=0.01, refractory_us=100,
                        capacity=8 * 1280 * 720, th_pos_uniform=0.15, th_neg_uniform=0.15, t0=0,
                        tick=1000, max_dt=1000, order=1, validate=1, epoch=1)
    n = L.evs_step_workspace_bytes(ctypes.byref(p))
    assert n > 8 * 1280 * 720 * 8  # holds the pixel-major key scratch
    p.width = 70000
    assert L.evs_step_workspace_bytes(ctypes.byref(p)) == 0  # uint16 coordinates


def test_seed_pcg64_matches_numpy_golden():
    """evs_seed_pcg64 is a host function of the product library: numpy SeedSequence parity."""
    from paper_2602_15018_b200 import _lib

    L = _lib.load()
    g = np.load(os.path.join(ROOT, "tests", "golden", "pcg64.npz"))
    for s, st in zip(g["seeds"], g["states"]):
        seed = int(s)
        words = []
        while True:
            words.append(seed & 0xFFFFFFFF)
            seed >>= 32
            if seed == 0:
                break
        w = np.array(words, np.uint32)
        out = np.zeros(4, np.uint64)
        L.evs_seed_pcg64(w.ctypes.data, len(w), out.ctypes.data)
        assert np.array_equal(out, st), s
