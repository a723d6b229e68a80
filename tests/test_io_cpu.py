"""Host-side io layer (paper_2306_08252_b200/io.py) against the reference's own fixtures and
goldens generated from the reference (tests/golden/ref_io.npz, make_golden.py): loaders
(io/loaders.hpp), generators (io/synthetic.hpp), batching (io/batching.hpp).  CPU only."""
from pathlib import Path

import numpy as np
import pytest

from paper_2306_08252_b200 import DataError
from paper_2306_08252_b200 import io as dio
from tests.golden.make_golden import IO_BATCHES, IO_SYNTH

GOLD = Path(__file__).resolve().parent / "golden"

# the three micro graphs of proj/tests/fixtures/*.mtx and their golden/*.csr dumps
TINY = "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2\n"
TRIANGLE = ("%%MatrixMarket matrix coordinate real general\n% a directed 3-cycle with edge weights\n"
            "3 3 3\n1 2 1.5\n2 3 2.5\n3 1 3.5\n")
STAR = ("%%MatrixMarket matrix coordinate pattern symmetric\n% hub-and-spoke graph stored as a lower triangle\n"
        "5 5 4\n2 1\n3 1\n4 1\n5 1\n")


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_mt19937_64_is_the_std_generator():
    # 10000th output of a default-seeded std::mt19937_64 (C++ standard, [rand.predef])
    g = dio.Mt19937_64(5489)
    assert int(g.draw(10000)[-1]) == 9981545732273789042
    z = np.load(GOLD / "synth_uniform_beef.npz")
    s, d = dio.synth_uniform_pairs(65536, 1000000, 0xBEEF)   # acceptance_test.cpp:241
    assert np.array_equal(s[:64], z["head_src"]) and np.array_equal(d[:64], z["head_dst"])
    assert s.astype(np.uint64).sum() == z["sum_src"] and d.astype(np.uint64).sum() == z["sum_dst"]
    assert np.bitwise_xor.reduce(s) == z["xor_src"] and np.bitwise_xor.reduce(d) == z["xor_dst"]


def test_matrix_market_golden_csr_dumps(tmp_path):
    # io_test.cpp:60-80 + fixtures/golden/*.csr
    c = dio.load_matrix_market(_write(tmp_path, "tiny.mtx", TINY))
    assert c.vertex_count == 2 and list(c.offsets) == [0, 1, 1] and list(c.destinations) == [1]
    assert dio.write_csr(c) == "vertices 2\nedges 1\noffsets 0 1 1\ndestinations 1\n"
    c = dio.load_matrix_market(_write(tmp_path, "tiny.mtx", TINY), symmetrize=True)
    assert list(c.offsets) == [0, 1, 2] and list(c.destinations) == [1, 0]
    c = dio.load_matrix_market(_write(tmp_path, "tri.mtx", TRIANGLE))
    assert dio.write_csr(c) == "vertices 3\nedges 3\noffsets 0 1 2 3\ndestinations 1 2 0\n"
    c = dio.load_matrix_market(_write(tmp_path, "star.mtx", STAR), symmetrize=True)
    assert dio.write_csr(c) == "vertices 5\nedges 8\noffsets 0 4 5 6 7 8\ndestinations 1 2 3 4 0 0 0 0\n"


@pytest.mark.parametrize("content,needle", [
    ("%%MatrixMarket matrix array real general\n2 2\n", "coordinate"),
    ("not a header\n", "line 1"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 x\n", "line 3"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1.5\n", "not a non-negative integer"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n", "outside the declared"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n", "declared 2 entries"),
])
def test_matrix_market_parse_errors_carry_line_numbers(tmp_path, content, needle):
    # io_test.cpp:82-108
    with pytest.raises(DataError, match=needle):
        dio.load_matrix_market(_write(tmp_path, "bad.mtx", content))


def test_edge_list_loader(tmp_path):
    # io_test.cpp:110-137
    p = _write(tmp_path, "g.el", "# comment\n0 2\n2 1\n\n2 0\n")
    c = dio.load_edge_list(p)
    assert c.vertex_count == 3 and list(c.offsets) == [0, 1, 1, 3] and list(c.destinations) == [2, 1, 0]
    assert dio.load_edge_list(p, True).edge_count() == 6
    with pytest.raises(DataError, match="line 2"):
        dio.load_edge_list(_write(tmp_path, "bad.el", "0 1\n1 -2\n"))
    e = dio.load_edge_list(_write(tmp_path, "empty.el", ""))
    assert e.vertex_count == 0 and e.edge_count() == 0
    with pytest.raises(DataError, match="cannot open"):
        dio.load_edge_list(str(tmp_path / "missing.el"))


def test_synthetic_generators_match_reference_golden():
    z = np.load(GOLD / "ref_io.npz")
    for i, (kind, v, e, seed) in enumerate(IO_SYNTH):
        c = dio.synth_uniform(v, e, seed) if kind == 0 else dio.synth_power_law(v, e, seed)
        assert np.array_equal(c.offsets, z[f"synth{i}_off"]), (i, "offsets")
        assert np.array_equal(c.destinations, z[f"synth{i}_dst"]), (i, "destinations")
    with pytest.raises(DataError):
        dio.synth_uniform(0, 10, 1)


def test_make_batches_match_reference_golden():
    z = np.load(GOLD / "ref_io.npz")
    for i, (si, batch, _, shuffled, seed) in enumerate(IO_BATCHES):
        kind, v, e, sseed = IO_SYNTH[si]
        csr = dio.Csr(v, z[f"synth{si}_off"], z[f"synth{si}_dst"])
        bs = dio.make_batches(csr, batch, order=dio.EdgeOrder.Shuffled if shuffled else dio.EdgeOrder.Prefix, seed=seed)
        assert [b.edge_count() for b in bs] == list(z[f"batch{i}_sizes"]), i
        src = np.concatenate([dio.edge_sequence(dio.Csr(v, b.offsets, b.destinations))[0] for b in bs])
        dst = np.concatenate([b.destinations for b in bs])
        assert np.array_equal(src, z[f"batch{i}_src"]) and np.array_equal(dst, z[f"batch{i}_dst"]), i
        for b in bs:   # io_test.cpp:139-204: every batch spans the full vertex count
            assert b.offsets.size == v + 1
    # bulk batch of an empty graph still yields one (empty) batch
    assert len(dio.make_batches(dio.Csr(3, np.zeros(4, np.uint64), np.zeros(0, np.uint32)), 5)) == 1


def test_io_against_live_reference_when_present():
    """Where oracle/_ref exists (the build container) the generators are also checked at sizes the
    fixtures do not hold."""
    import ctypes as C
    from tests.drivers import load_ref
    ref = load_ref()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    for kind, v, e, seed in [(0, 1000, 30000, 99), (1, 3000, 50000, 123)]:
        off = np.zeros(v + 1, np.uint64); dst = np.zeros(e, np.uint32)
        assert ref.ref_synth_csr(kind, C.c_uint64(v), C.c_uint64(e), C.c_uint64(seed), C.c_void_p(off.ctypes.data),
                                 C.c_void_p(dst.ctypes.data)) == 0
        c = dio.synth_uniform(v, e, seed) if kind == 0 else dio.synth_power_law(v, e, seed)
        assert np.array_equal(c.offsets, off) and np.array_equal(c.destinations, dst)
