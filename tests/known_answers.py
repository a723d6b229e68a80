"""Known-answer cases of the reference's own tests, restated as op scripts.

Each entry cites the reference test it restates (semantic, layout-free part
only: SURVEY.md §8c).  The same scripts run against the oracle restatement,
the real reference (oracle/_ref) and the CUDA path.
"""
import numpy as np


def u32(*xs):
    return np.asarray(xs, dtype=np.uint32)


def pairs(*ps):
    return u32(*[p[0] for p in ps]), u32(*[p[1] for p in ps])


SMALL = {"arena_bytes": 1 << 20, "initial_fraction": 0.5, "reclaim": True}


def _q(*ps):
    s, d = pairs(*ps)
    return ("query", s, d)


KNOWN_ANSWER_SCRIPTS = [
    # proj/tests/batch_engine_test.cpp:305-312 DeleteBatch.OneDeleteEntryRemovesAllCopies
    ("delete_removes_all_copies", {**SMALL, "v0": 4, "block_size": 4}, [
        ("insert", *pairs((1, 2), (1, 2), (1, 3))),
        ("delete", *pairs((1, 2))),
        ("check",), _q((1, 2), (1, 3)),
    ]),
    # :280-288 DeleteBatch.AbsentEdgeIsANoop
    ("absent_edge_noop", {**SMALL, "v0": 4, "block_size": 4}, [
        ("insert", *pairs((1, 2), (1, 3))),
        ("delete", *pairs((2, 3), (1, 0))),
        ("check",), _q((1, 2), (1, 3), (2, 3), (1, 0)),
    ]),
    # :290-297 DeleteBatch.TombstonesSingleMatch (query/degree part)
    ("single_match", {**SMALL, "v0": 4, "block_size": 4}, [
        ("insert", *pairs((1, 2), (1, 3))),
        ("delete", *pairs((1, 2))),
        ("check",), _q((1, 2), (1, 3)),
    ]),
    # :343-373 DeleteBatch.ReclaimReturnsEmptyTailBlocks (observable part)
    ("reclaim_tail", {**SMALL, "v0": 2, "block_size": 2}, [
        ("insert", *pairs((0, 0), (0, 0), (0, 0), (0, 1), (0, 1), (0, 1))),
        ("delete", *pairs((0, 1))), ("check",),
        ("delete", *pairs((0, 0))), ("check",),
        ("insert", *pairs((0, 1))), ("check",), _q((0, 1), (0, 0)),
    ]),
    # :375-388 DeleteBatch.NoReclaimKeepsBlocksInPlace
    ("no_reclaim", {**SMALL, "reclaim": False, "v0": 2, "block_size": 2}, [
        ("insert", *pairs((0, 1), (0, 1), (0, 1), (0, 1))),
        ("delete", *pairs((0, 1))), ("check",), _q((0, 1)),
    ]),
    # :390-413 QueryEdge.*
    ("query_semantics", {**SMALL, "v0": 4, "block_size": 4}, [
        _q((0, 1)),
        ("insert", *pairs((1, 2))),
        _q((1, 2), (1, 3), (2, 1), (7, 0)),
        ("del_vertices", u32(1)),
        _q((1, 2)),
    ]),
    # :270-278 InsertBatch.RetiredSourceRejected
    ("retired_source_rejected", {**SMALL, "v0": 4, "block_size": 4}, [
        ("del_vertices", u32(1)),
        ("insert", *pairs((1, 0))),           # DataError, graph untouched
        ("insert", *pairs((0, 1))),
        ("check",),
    ]),
    # :116-148 PlanBatch.MalformedCsrRejected (CSR entry point)
    ("malformed_csr", {**SMALL, "v0": 4, "block_size": 4}, [
        ("insert_csr", np.asarray([0, 1, 1], np.uint64), u32(0)),
        ("insert_csr", np.asarray([0, 2, 1, 2, 2], np.uint64), u32(0, 1)),
        ("insert_csr", np.asarray([1, 1, 1, 1, 1], np.uint64), u32(0)),
        ("insert_csr", np.asarray([0, 1, 1, 1, 1], np.uint64), u32(4)),
        ("insert_csr", np.asarray([0, 1, 1, 1, 2], np.uint64), u32(0)),
        ("delete_csr", np.asarray([0, 1, 1, 1, 1], np.uint64), u32(4)),   # deletes are range-checked too (graph.hpp:199)
        ("check",),
        ("insert_csr", np.asarray([0, 1, 1, 2, 2], np.uint64), u32(3, 0)),
        ("check",),
    ]),
    # :159-173 InsertBatch.FreshVertexSixEdgesTwoBlocks + :194-210 resume at last-insert
    ("resume_at_last_insert", {**SMALL, "v0": 2, "block_size": 4}, [
        ("insert", *pairs(*[(0, 1)] * 6)), ("check",),
        ("insert", *pairs(*[(0, 0)] * 10)), ("check",), _q((0, 1), (0, 0), (1, 0)),
    ]),
    # :437-468 InsertVertices.*  (453 -> 512 -> 513/1024)
    ("insert_vertices_capacity", {**SMALL, "v0": 453, "block_size": 4}, [
        ("check",), ("add_vertices", 59), ("check",), ("add_vertices", 1), ("check",),
        ("add_vertices", 0), ("check",),
    ]),
    # :470-497 DeleteVertices.* (skipped ids in encounter order, in-call duplicates)
    ("delete_vertices_skipped", {**SMALL, "v0": 4, "block_size": 4}, [
        ("insert", *pairs((1, 2), (1, 3))),
        ("del_vertices", u32(1)), ("check",), _q((1, 2)),
        ("del_vertices", u32(2, 9, 2)), ("check",),
    ]),
    # :499-514 DeleteVertices.RetiredIdStaysDeadAndNewIdsStartFresh
    ("retired_id_stays_dead", {**SMALL, "v0": 2, "block_size": 4}, [
        ("insert", *pairs((1, 0))),
        ("del_vertices", u32(1)),
        ("add_vertices", 1),
        ("insert", *pairs((2, 0))),
        ("check",), _q((2, 0), (1, 0)),
    ]),
    # proj/tests/oracle_test.cpp:24-31 multiset delete; :33-45 dead source deletes ignored
    ("dead_source_delete_ignored", {**SMALL, "v0": 4, "block_size": 3}, [
        ("insert", *pairs((0, 1), (0, 1), (2, 3), (2, 3), (2, 1))),
        ("del_vertices", u32(2)),
        ("delete", *pairs((2, 3), (0, 1))),
        ("check",), _q((0, 1), (2, 3), (2, 1)),
    ]),
    # vertex delete without reclaim keeps the sentinel count (graph.hpp:264-272)
    ("dead_vertex_no_reclaim_keeps_degree", {**SMALL, "reclaim": False, "v0": 4, "block_size": 2}, [
        ("insert", *pairs((3, 0), (3, 1), (3, 2), (0, 3))),
        ("del_vertices", u32(3)), ("check",), _q((3, 0), (0, 3)),
    ]),
    # golden micro-graph: proj/tests/fixtures/golden/star_symmetric.csr (offsets 0 4 5 6 7 8)
    ("star_symmetric_golden", {**SMALL, "v0": 5, "block_size": 2}, [
        ("insert_csr", np.asarray([0, 4, 5, 6, 7, 8], np.uint64), u32(1, 2, 3, 4, 0, 0, 0, 0)),
        ("check",), _q((0, 1), (0, 4), (4, 0), (1, 2)),
    ]),
    # proj/tests/fixtures/golden/triangle_weighted.csr + tiny_directed.csr
    ("triangle_golden", {**SMALL, "v0": 3, "block_size": 1}, [
        ("insert_csr", np.asarray([0, 1, 2, 3], np.uint64), u32(1, 2, 0)),
        ("check",), _q((0, 1), (1, 2), (2, 0), (0, 2)),
        ("delete_csr", np.asarray([0, 1, 1, 2], np.uint64), u32(1, 0)),
        ("check",),
    ]),
    # empty batches change nothing (batch_engine_test.cpp:150-157)
    ("empty_batches", {**SMALL, "v0": 4, "block_size": 4}, [
        ("insert", u32(), u32()), ("delete", u32(), u32()),
        ("insert_csr", np.asarray([0, 0, 0, 0, 0], np.uint64), u32()),
        ("check",),
    ]),
]
