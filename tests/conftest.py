"""Shared test setup: markers, golden-fixture access, oracle handle."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@pytest.fixture
def native_options():
    """Set library path overrides (eg_set_option) for one test; reset after."""
    from paper_0904_3151_b200 import _native

    def set_options(**kw):
        for k, v in kw.items():
            _native.check(_native.lib().eg_set_option(k.encode(), int(v)), f"option {k}")
    yield set_options
    _native.lib().eg_reset_options()


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc
    orc.build()
    return orc


FIG2_STRINGS = [
    "1011111100111110", "1101011101110001", "1100100011011100",
    "0100000101111101", "1010001011101010", "1111001110010111",
    "0000000100111110", "0101100101111000", "1101100011011110",
    "1001001110010111",
]
FIG2_CLOSE_PAIRS = {(2, 8), (5, 9)}


def bits_from_strings(strings):
    return np.array([[int(c) for c in s] for s in strings], dtype=np.uint8)


def pack_bits(bits):
    """Little-endian packing: bit t -> word t//64, position t%64."""
    bits = np.asarray(bits, dtype=np.uint8)
    n, length = bits.shape
    W = max(1, -(-length // 64))
    packed = np.packbits(bits, axis=1, bitorder="little")
    buf = np.zeros((n, W * 8), dtype=np.uint8)
    buf[:, :packed.shape[1]] = packed
    return buf.view("<u8").copy()
