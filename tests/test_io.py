"""Edge-list files (reference io.py:122-195): GPU formatting of write_edges
against bytes written by the reference itself (tests/golden/io_edges.npz,
made by make_golden.py), the host parser, and the reference's own cases
(tests/test_io.py of the reference, restated)."""

import numpy as np
import pytest

from conftest import golden


# ----------------------------------------------------------- host (no GPU)
def test_read_edges_parses_reference_bytes(tmp_path, manifest):
    from paper_0904_3151_b200 import read_edges
    g = golden("io_edges")
    path = tmp_path / "e.txt"
    path.write_bytes(g["text"].tobytes())
    edges, meta = read_edges(path)
    np.testing.assert_array_equal(edges.pairs, g["pairs"])
    # %.9f text: the parsed distance is within half a unit of the 9th digit
    assert np.all(np.abs(edges.distances - g["dist"]) <= 5e-10 * (1 + 1e-9) + 1e-15 * g["dist"])
    assert meta == manifest["io_edges"]["meta"]


@pytest.mark.parametrize("body", [
    "1 0 0.5\n",                  # i >= j
    "0 1 0.5\n0 1 0.5\n",         # duplicate
    "1 2 0.5\n0 1 0.5\n",         # out of order
    "0 1\n",                      # missing column
    "0 x 0.5\n",                  # not an integer
])
def test_read_edges_rejects_malformed(tmp_path, body):
    from paper_0904_3151_b200 import DataError, read_edges
    path = tmp_path / "e.txt"
    path.write_text("# nodes=3\n" + body)
    with pytest.raises(DataError):
        read_edges(path)


def test_read_edges_error_lines(tmp_path):
    from paper_0904_3151_b200 import DataError, read_edges
    path = tmp_path / "e.txt"
    path.write_text("# nodes=9\n0 1 0.5\n\n2 3 0.1\n3 3 0.2\n")
    with pytest.raises(DataError, match=r":5: need 0 <= i < j"):
        read_edges(path)
    path.write_text("0 1 0.5\n2 3 0.1\n2 3 0.2\n")
    with pytest.raises(DataError, match=r":3: pairs must be sorted and unique"):
        read_edges(path)


# ------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def eg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_0904_3151_b200 as eg
    return eg


@pytest.mark.gpu
def test_write_edges_bytes_equal_reference(eg, tmp_path, manifest):
    g = golden("io_edges")
    path = tmp_path / "e.txt"
    eg.write_edges(path, eg.EdgeList(g["pairs"], g["dist"]), manifest["io_edges"]["meta"])
    assert path.read_bytes() == g["text"].tobytes()


@pytest.mark.gpu
def test_write_edges_from_device_and_round_trip(eg, tmp_path):
    import torch
    from paper_0904_3151_b200 import workloads
    x = workloads.cfg1_points(3_000, clusters=60)
    params = eg.MsmParams(epsilon=0.1, gamma=1e-6, length=32, mismatch=2, blocks=8,
                          replicates=1, seed=0)
    out = eg.build_graph_device(torch.from_numpy(x).cuda(), params)
    p1, p2 = tmp_path / "a.txt", tmp_path / "b.txt"
    eg.write_edges(p1, (out["keys"], out["dist"]), {"nodes": 3000})
    g = eg.build_graph(x, params)
    eg.write_edges(p2, g.edge_list, {"nodes": 3000})
    assert p1.read_bytes() == p2.read_bytes()
    back, meta = eg.read_edges(p1)
    np.testing.assert_array_equal(back.pairs, g.edge_list.pairs)
    assert meta == {"nodes": 3000}
    # the stable-format case of the reference's tests
    p3 = tmp_path / "c.txt"
    eg.write_edges(p3, eg.EdgeList.from_rows([(0, 1, 0.123456789123)]), {"nodes": 2})
    assert p3.read_text() == "# nodes=2\n0 1 0.123456789\n"
    eg.write_edges(p3, eg.EdgeList(), {"nodes": 0})
    back, meta = eg.read_edges(p3)
    assert len(back) == 0 and meta["nodes"] == 0


@pytest.mark.gpu
def test_write_edges_random_doubles_match_python_format(eg, tmp_path):
    """%.9f of arbitrary doubles (all exponents that fit, ties at the 9th
    digit) equals Python's correctly rounded formatting."""
    rng = np.random.default_rng(8)
    d = np.concatenate([rng.random(3000) * 2, 10.0 ** rng.uniform(-12, 9, 3000),
                        (rng.integers(0, 2 ** 20, 2000) + 0.5) / 1e9,      # exact-ish ties
                        np.ldexp(rng.integers(1, 2 ** 30, 2000).astype(np.float64), -31)])
    pairs = np.stack([np.arange(d.size), np.arange(d.size) + 1], axis=1)
    path = tmp_path / "r.txt"
    eg.write_edges(path, eg.EdgeList(pairs, d))
    want = "".join(f"{i} {j} {v:.9f}\n" for (i, j), v in zip(pairs.tolist(), d.tolist()))
    assert path.read_text() == want


# --------------------------------------------------------------- datasets
def test_dataset_round_trip_and_reference_bytes(tmp_path):
    """write_dataset bytes = the reference's header + float32 payload;
    read_dataset returns the rows (reference tests/test_io.py cases)."""
    import struct
    from paper_0904_3151_b200 import read_dataset, write_dataset
    rng = np.random.default_rng(1)
    data = rng.standard_normal((37, 5)).astype(np.float32)
    path = tmp_path / "d.bin"
    write_dataset(path, data)
    raw = path.read_bytes()
    assert raw[:28] == struct.pack("<4sIQQI", b"EPGD", 1, 37, 5, 4)
    assert raw[28:] == data.astype("<f4").tobytes()
    np.testing.assert_array_equal(read_dataset(path).vectors, data)


def test_dataset_csv_fallback_and_errors(tmp_path):
    from paper_0904_3151_b200 import DataError, read_dataset, write_dataset
    path = tmp_path / "d.csv"
    path.write_text("1.5,2.0\n-0.25,3.0\n0.125,7.0\n")
    back = read_dataset(path)
    assert back.vectors.dtype == np.float32
    np.testing.assert_array_equal(back.vectors, np.array([[1.5, 2.0], [-0.25, 3.0],
                                                          [0.125, 7.0]], dtype=np.float32))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"not a dataset at all")
    with pytest.raises(DataError):
        read_dataset(bad)
    d = tmp_path / "t.bin"
    write_dataset(d, np.ones((20, 4), np.float32))
    d.write_bytes(d.read_bytes()[:-8])
    with pytest.raises(DataError, match="payload"):
        read_dataset(d)
    with pytest.raises(DataError):
        write_dataset(tmp_path / "n.bin", np.array([[1.0, np.nan]], dtype=np.float32))


@pytest.mark.gpu
def test_read_dataset_device(eg, tmp_path):
    rng = np.random.default_rng(4)
    data = rng.standard_normal((1000, 48)).astype(np.float32)
    path = tmp_path / "d.bin"
    eg.write_dataset(path, data)
    x = eg.read_dataset_device(path)
    assert x.is_cuda and x.dtype.is_floating_point
    np.testing.assert_array_equal(x.cpu().numpy(), data)
    # a corrupted payload value is caught on the device
    raw = bytearray(path.read_bytes())
    raw[28 + 4 * 777:28 + 4 * 778] = np.array([np.inf], dtype="<f4").tobytes()
    path.write_bytes(bytes(raw))
    with pytest.raises(eg.DataError, match="non-finite"):
        eg.read_dataset_device(path)


@pytest.mark.gpu
def test_write_edges_chunked_equals_single_call(eg, tmp_path, monkeypatch):
    """Edge lists longer than one eg_format_edges call are written in chunks
    with identical bytes (chunk size forced small)."""
    g = golden("io_edges")
    edges = eg.EdgeList(g["pairs"], g["dist"])
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    eg.write_edges(a, edges, {"nodes": 7})
    from paper_0904_3151_b200 import io as egio
    monkeypatch.setattr(egio, "FORMAT_CHUNK", 997)
    eg.write_edges(b, edges, {"nodes": 7})
    assert a.read_bytes() == b.read_bytes()


# ------------------------------------------------------------------ pools
@pytest.mark.parametrize("length", [1, 7, 60, 64, 65, 128, 130])
def test_pool_round_trip_and_reference_bytes(tmp_path, length):
    import struct
    from paper_0904_3151_b200 import BitStringPool, read_pool, write_pool
    rng = np.random.default_rng(length)
    bits = (rng.random((9, length)) < 0.5).astype(np.uint8)
    pool = BitStringPool.from_bits(bits)
    path = tmp_path / "p.bin"
    write_pool(path, pool)
    raw = path.read_bytes()
    row_bytes = -(-length // 8)
    assert raw[:24] == struct.pack("<4sIQQ", b"EPGP", 1, 9, length)
    assert len(raw) == 24 + 9 * row_bytes
    # byte b of a row holds bits 8b..8b+7, bit t at position t % 8
    packed = np.packbits(bits, axis=1, bitorder="little")
    assert raw[24:] == packed.tobytes()
    back = read_pool(path)
    assert back.length == length
    np.testing.assert_array_equal(back.words, pool.words)


def test_pool_rejects_padding_and_magic(tmp_path):
    from paper_0904_3151_b200 import BitStringPool, DataError, read_pool, write_pool
    rng = np.random.default_rng(5)
    pool = BitStringPool.from_bits((rng.random((4, 60)) < 0.5).astype(np.uint8))
    path = tmp_path / "p.bin"
    write_pool(path, pool)
    raw = bytearray(path.read_bytes())
    raw[-1] |= 0xF0
    path.write_bytes(bytes(raw))
    with pytest.raises(DataError, match="padding"):
        read_pool(path)
    path.write_bytes(b"EPGX" + b"\x00" * 40)
    with pytest.raises(DataError):
        read_pool(path)
