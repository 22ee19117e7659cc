"""CPU tests of the product boundary: the C-ABI library loads, exports every
symbol include/hmgp_cuda.h declares, and its host-only utilities (input
generators, defaults) agree with the oracle bit-for-bit.  No GPU calls."""
import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "hmgp_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hmgp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(hm):
    lib = ctypes.CDLL(hm.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    import subprocess
    from paper_2104_07146_b200 import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_generators_match_oracle(hm, oracle):
    assert np.array_equal(hm.jittered_grid(64, 1), oracle.jittered_grid(64, 1))
    assert np.array_equal(hm.random_locations(1000, 42), oracle.random_locations(1000, 42))
    assert np.array_equal(hm.random_locations(999, 5, dim=3), oracle.random_locations(999, 5, dim=3))
    assert np.array_equal(hm.normals(5000, 17), oracle.normals(5000, 17))
    g = hm.jittered_grid(8, 3)
    cell = np.floor(g * 8).astype(int)  # every point stays inside its cell
    assert np.array_equal(cell[:, 0], np.repeat(np.arange(8), 8))
    assert np.array_equal(cell[:, 1], np.tile(np.arange(8), 8))


def test_default_config_matches_reference():
    from paper_2104_07146_b200 import HConfig, _Config, _lib
    c = _Config()
    _lib.hmgp_default_config(ctypes.byref(c))
    assert (c.eta, c.leaf_size, c.rank.mode, c.rank.eps, c.rank.max_rank, c.eps_factor, c.form) == (
        2.0, 32, 0, 1e-6, 256, -1.0, 1)
    assert HConfig().factor_eps() == 1e-6
