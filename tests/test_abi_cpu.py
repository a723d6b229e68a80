"""The C-ABI library loads without a GPU and exports every symbol the header declares."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dyngraph_b200.h"


def _declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", text)))


def test_header_cites_reference_lines():
    text = HEADER.read_text()
    for needle in ("graph.hpp:167-188", "graph.hpp:195-222", "graph.hpp:228-241", "graph.hpp:252-276",
                   "csr.hpp:49-73", "vertex_dictionary.hpp:53-71", "block_pool.hpp:99-116"):
        assert needle in text, needle


def test_library_exports_every_declared_symbol():
    from paper_2306_08252_b200 import _lib
    from paper_2306_08252_b200.build import build_library
    build_library()
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), f"{n} declared in the header but not exported"
        assert n in _lib.SIGNATURES, f"{n} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(names), set(_lib.SIGNATURES) ^ set(names)
    assert lib.dg_abi_version() == 1


def test_owner_permutation_is_a_bijection():
    from paper_2306_08252_b200 import _lib
    lib = _lib.load()
    for bits in (1, 4, 11, 16):
        img = {lib.dg_owner_perm(v, bits) for v in range(1 << bits)}
        assert img == set(range(1 << bits))
    rng = np.random.default_rng(0)
    for bits in (22, 26, 32):
        for v in rng.integers(0, 1 << bits, 2000):
            p = lib.dg_owner_perm(int(v), bits)
            assert p < (1 << bits) and lib.dg_owner_perm_inv(p, bits) == int(v)
    # R-MAT-style skew (sources sharing low bits) spreads evenly over 8 owners
    hot = np.arange(0, 1 << 22, 8, dtype=np.uint64)[:40000]
    owners = np.array([lib.dg_owner_perm(int(v), 22) % 8 for v in hot])
    share = np.bincount(owners, minlength=8) / len(owners)
    assert share.max() < 0.15


def test_missing_library_fails_loudly(tmp_path):
    from paper_2306_08252_b200 import _lib
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load(tmp_path / "nope.so")


def test_host_side_csr_helpers():
    from paper_2306_08252_b200 import BatchKind, compute_block_size, csr_from_pairs, DataError
    b = csr_from_pairs(BatchKind.Insert, 4, [2, 0, 2, 2], [1, 3, 0, 1])
    assert list(b.offsets) == [0, 1, 1, 4, 4] and list(b.destinations) == [3, 1, 0, 1]  # stable (csr.hpp:29-45)
    assert compute_block_size(b) == 2  # 4 edges / 2 sources
    # batch_engine_test.cpp:36-82 block-size rule: round half up, min 1
    assert compute_block_size(csr_from_pairs(BatchKind.Insert, 4, [0, 0, 0, 1, 2], [0] * 5)) == 2  # 5/3 = 1.67
    assert compute_block_size(csr_from_pairs(BatchKind.Insert, 4, [0, 0, 0, 1], [0] * 4)) == 2      # 4/2
    assert compute_block_size(csr_from_pairs(BatchKind.Insert, 4, [0, 0, 0, 1, 1, 2, 3], [0] * 7)) == 2  # 1.75
    with pytest.raises(DataError):
        compute_block_size(csr_from_pairs(BatchKind.Insert, 4, [], []))
    with pytest.raises(DataError):
        csr_from_pairs(BatchKind.Insert, 4, [4], [0])


def test_cpp_mirror_header_compiles_standalone(tmp_path):
    """include/dyngraph_b200.hpp (the C++ mirror of dyngraph::DynamicGraph) needs only a C++17 compiler."""
    import subprocess
    src = tmp_path / "t.cpp"
    src.write_text('#include "dyngraph_b200.hpp"\n'
                   "int main() { dyngraph_b200::CsrBatch b = dyngraph_b200::csr_from_pairs("
                   "dyngraph_b200::BatchKind::Insert, 3, {{2, 1}, {0, 2}, {2, 0}});\n"
                   "  return (b.offsets == std::vector<std::uint64_t>{0, 1, 1, 3} && "
                   "b.destinations == std::vector<std::uint32_t>{2, 1, 0}) ? 0 : 1; }\n")
    exe = tmp_path / "t"
    from paper_2306_08252_b200.build import LIB_PATH, build_library
    build_library()
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", str(src), "-o", str(exe),
                    f"-L{LIB_PATH.parent}", "-ldyngraph_b200", f"-Wl,-rpath,{LIB_PATH.parent}"], check=True)
    assert subprocess.run([str(exe)]).returncode == 0


def test_ctypes_signatures_match_header_arity():
    """Every ctypes signature has as many arguments as the header's prototype (a missing one
    shifts every later pointer)."""
    from paper_2306_08252_b200 import _lib
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    protos = dict(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", text))
    assert len(protos) >= 30
    for name, args in protos.items():
        args = args.strip()
        n = 0 if args in ("", "void") else args.count(",") + 1
        assert len(_lib.SIGNATURES[name][1]) == n, (name, n, len(_lib.SIGNATURES[name][1]))
