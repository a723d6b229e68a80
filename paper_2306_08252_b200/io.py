"""Host-side callers and data formats either side of the hot path:
the reference's `io/` layer restated over the GPU store.

  loaders      load_matrix_market / load_edge_list / write_csr   (io/loaders.hpp:72-176)
  generators   synth_uniform / synth_power_law                    (io/synthetic.hpp:16-66)
  batching     make_batches (prefix or Fisher-Yates-shuffled)      (io/batching.hpp:46-66)
  runner       WorkloadSpec / run_workload / RunReport / write_csv (io/workload.hpp:22-208)

Everything here is host preprocessing or orchestration; the graph operations go
through `DynamicGraph` (the C ABI).  Same names, argument meaning and error
behaviour as the reference (DataError with line numbers for parse errors).
The random streams are the reference's: std::mt19937_64 draws, `rng() % n`.

Draw order: the reference builds pairs with `emplace_back(rng() % V, rng() % V)`
(io/synthetic.hpp:23-24, :62; io/workload.hpp:173-174).  C++ leaves the order of
the two draws unspecified and g++ — the toolchain the reference is built with —
evaluates the arguments right to left, so the FIRST draw of every pair is the
destination.  This module follows the reference AS BUILT (pinned by goldens
generated from the compiled reference, tests/golden/ref_io.npz).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, List, Optional

import numpy as np

from .csr import BatchKind, CsrBatch, compute_block_size
from .errors import DataError
from .graph import DynamicGraph, GraphConfig


# ---------------------------------------------------------------------------
# std::mt19937_64 (the reference's generator: io/synthetic.hpp:19, io/batching.hpp:33)
# ---------------------------------------------------------------------------
class Mt19937_64:
    """Bit-exact std::mt19937_64; the twist is vectorised over the 312-word state."""
    NN, MM = 312, 156
    UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)

    def __init__(self, seed: int):
        mt = np.zeros(self.NN, np.uint64)
        x = seed & 0xFFFFFFFFFFFFFFFF
        mt[0] = x
        for i in range(1, self.NN):
            x = (6364136223846793005 * (x ^ (x >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
            mt[i] = x
        self.mt = mt
        self.buf = np.zeros(0, np.uint64)
        self.pos = 0

    def _twist(self):
        mt, NN, MM = self.mt, self.NN, self.MM
        one = np.uint64(1)

        def mag(x):
            return np.where((x & one).astype(bool), self.MATRIX_A, np.uint64(0))
        # i in [0, NN-MM): uses old mt[i+1] and old mt[i+MM]
        x = (mt[0:NN - MM] & self.UM) | (mt[1:NN - MM + 1] & self.LM)
        mt[0:NN - MM] = mt[MM:NN] ^ (x >> one) ^ mag(x)
        # i in [NN-MM, NN-1): uses old mt[i+1] and NEW mt[i+MM-NN]
        x = (mt[NN - MM:NN - 1] & self.UM) | (mt[NN - MM + 1:NN] & self.LM)
        mt[NN - MM:NN - 1] = mt[0:MM - 1] ^ (x >> one) ^ mag(x)
        x = (mt[NN - 1] & self.UM) | (mt[0] & self.LM)
        mt[NN - 1] = mt[MM - 1] ^ (x >> one) ^ (self.MATRIX_A if int(x) & 1 else np.uint64(0))
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def draw(self, n: int) -> np.ndarray:
        """The next n outputs (uint64)."""
        out = np.empty(n, np.uint64)
        k = 0
        while k < n:
            if self.pos == self.buf.size:
                self.buf = self._twist()
                self.pos = 0
            take = min(n - k, self.buf.size - self.pos)
            out[k:k + take] = self.buf[self.pos:self.pos + take]
            self.pos += take
            k += take
        return out

    def __call__(self) -> int:
        return int(self.draw(1)[0])


# ---------------------------------------------------------------------------
# loaders (io/loaders.hpp)
# ---------------------------------------------------------------------------
@dataclass
class Csr:
    """A fully loaded graph in CSR form (io/loaders.hpp:18-25)."""
    vertex_count: int = 0
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    destinations: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def edge_count(self) -> int:
        return int(self.destinations.size)


def csr_from_edges(vertex_count: int, src, dst) -> Csr:
    """Stable counting sort by source (io/loaders.hpp:54-68)."""
    src = np.asarray(src, np.uint32)
    dst = np.asarray(dst, np.uint32)
    counts = np.bincount(src, minlength=vertex_count) if src.size else np.zeros(vertex_count, np.int64)
    offsets = np.zeros(vertex_count + 1, np.uint64)
    np.cumsum(counts, out=offsets[1:])
    order = np.argsort(src, kind="stable")
    return Csr(vertex_count, offsets, dst[order].astype(np.uint32))


def _split_ws(line: str) -> List[str]:
    return [t for t in line.replace("\t", " ").replace("\r", " ").split(" ") if t]


def _parse_id(token: str, line_no: int, what: str) -> int:
    # std::from_chars on an unsigned integer: digits only, the whole token
    if not token.isascii() or not token.isdigit():
        raise DataError(f"line {line_no}: {what} '{token}' is not a non-negative integer")
    return int(token)


def load_matrix_market(path: str, symmetrize: bool = False) -> Csr:
    """Matrix Market coordinate loader, 1-based ids (io/loaders.hpp:72-131)."""
    try:
        fh = open(path, "r")
    except OSError:
        raise DataError(f"cannot open '{path}'")
    with fh:
        lines = fh.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise DataError(f"{path}: empty file")
    header = _split_ws(lines[0])
    if len(header) < 4 or header[0] != "%%MatrixMarket" or header[1] != "matrix":
        raise DataError("line 1: expected a '%%MatrixMarket matrix' header")
    if header[2] != "coordinate":
        raise DataError("line 1: only the coordinate format is supported")
    rows = cols = declared = 0
    have_size = False
    src: List[int] = []
    dst: List[int] = []
    for line_no, line in enumerate(lines[1:], start=2):
        if line.startswith("%"):
            continue
        tokens = _split_ws(line)
        if not tokens:
            continue
        if not have_size:
            if len(tokens) < 3:
                raise DataError(f"line {line_no}: expected 'rows cols entries'")
            rows = _parse_id(tokens[0], line_no, "row count")
            cols = _parse_id(tokens[1], line_no, "column count")
            declared = _parse_id(tokens[2], line_no, "entry count")
            have_size = True
            continue
        if len(tokens) < 2:
            raise DataError(f"line {line_no}: expected 'row col [value]'")
        r = _parse_id(tokens[0], line_no, "row id")
        c = _parse_id(tokens[1], line_no, "column id")
        if r < 1 or r > rows or c < 1 or c > cols:
            raise DataError(f"line {line_no}: entry ({r}, {c}) is outside the declared {rows}x{cols} shape")
        src.append(r - 1)
        dst.append(c - 1)
        if symmetrize and r != c:
            src.append(c - 1)
            dst.append(r - 1)
    if not have_size:
        raise DataError(f"{path}: missing size line")
    if not symmetrize and len(src) != declared:
        raise DataError(f"{path}: declared {declared} entries, found {len(src)}")
    return csr_from_edges(max(rows, cols), src, dst)


def load_edge_list(path: str, symmetrize: bool = False) -> Csr:
    """'src dst' per line, 0-based, '#'/'%' comments (io/loaders.hpp:135-164)."""
    try:
        fh = open(path, "r")
    except OSError:
        raise DataError(f"cannot open '{path}'")
    with fh:
        lines = fh.read().split("\n")
    src: List[int] = []
    dst: List[int] = []
    max_id = 0
    for line_no, line in enumerate(lines, start=1):
        if line.startswith("#") or line.startswith("%"):
            continue
        tokens = _split_ws(line)
        if not tokens:
            continue
        if len(tokens) < 2:
            raise DataError(f"line {line_no}: expected 'src dst'")
        s = _parse_id(tokens[0], line_no, "source id")
        d = _parse_id(tokens[1], line_no, "destination id")
        max_id = max(max_id, s, d)
        src.append(s)
        dst.append(d)
        if symmetrize and s != d:
            src.append(d)
            dst.append(s)
    return csr_from_edges(max_id + 1 if src else 0, src, dst)


def write_csr(csr: Csr) -> str:
    """The plain-text CSR dump the reference's golden tests pin (io/loaders.hpp:167-176)."""
    return (f"vertices {csr.vertex_count}\n" f"edges {csr.edge_count()}\n"
            "offsets" + "".join(f" {int(o)}" for o in csr.offsets) + "\n"
            "destinations" + "".join(f" {int(d)}" for d in csr.destinations) + "\n")


# ---------------------------------------------------------------------------
# synthetic graphs (io/synthetic.hpp)
# ---------------------------------------------------------------------------
def synth_uniform_pairs(vertex_count: int, edge_count: int, seed: int):
    """(src, dst) in generation order (io/synthetic.hpp:19-25); per pair the destination is drawn
    first (see the module docstring)."""
    if vertex_count == 0:
        raise DataError("synthetic graph needs at least one vertex")
    r = Mt19937_64(seed).draw(2 * edge_count) % np.uint64(vertex_count)
    return r[1::2].astype(np.uint32), r[0::2].astype(np.uint32)


def synth_uniform(vertex_count: int, edge_count: int, seed: int) -> Csr:
    s, d = synth_uniform_pairs(vertex_count, edge_count, seed)
    return csr_from_edges(vertex_count, s, d)


def synth_power_law(vertex_count: int, edge_count: int, seed: int) -> Csr:
    """Sources by inverse CDF of the harmonic weights, uniform destinations (io/synthetic.hpp:32-66)."""
    if vertex_count == 0:
        raise DataError("synthetic graph needs at least one vertex")
    # the reference accumulates sequentially in double: np.cumsum does the same left-to-right sum
    cdf = np.cumsum(1.0 / np.arange(1, vertex_count + 1, dtype=np.float64))
    total = cdf[-1]
    r = Mt19937_64(seed).draw(2 * edge_count)
    dst = (r[0::2] % np.uint64(vertex_count)).astype(np.uint32)   # (drawn first, see the module docstring)
    u = (r[1::2] >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * total
    # first index with cdf[i] >= u, clamped to the last vertex (the reference's lo/hi search)
    src = np.minimum(np.searchsorted(cdf, u, side="left"), vertex_count - 1).astype(np.uint32)
    return csr_from_edges(vertex_count, src, dst)


# ---------------------------------------------------------------------------
# batching (io/batching.hpp)
# ---------------------------------------------------------------------------
class EdgeOrder(Enum):
    Prefix = 0
    Shuffled = 1


def edge_sequence(csr: Csr):
    src = np.repeat(np.arange(csr.vertex_count, dtype=np.uint32), np.diff(csr.offsets.astype(np.int64)))
    return src, csr.destinations.astype(np.uint32)


def deterministic_shuffle(n: int, seed: int) -> np.ndarray:
    """The permutation io/batching.hpp:31-37 applies: Fisher-Yates, j = rng() % i for i = n .. 2."""
    perm = np.arange(n, dtype=np.int64)
    if n > 1:
        draws = Mt19937_64(seed).draw(n - 1)
        for k, i in enumerate(range(n, 1, -1)):
            j = int(draws[k] % np.uint64(i))
            perm[i - 1], perm[j] = perm[j], perm[i - 1]
    return perm


def _batch_from_pairs(kind: BatchKind, vertex_count: int, s, d) -> CsrBatch:
    c = csr_from_edges(vertex_count, s, d)
    return CsrBatch(kind, c.offsets, c.destinations)


def make_batches(csr: Csr, batch_size: int, kind: BatchKind = BatchKind.Insert,
                 order: EdgeOrder = EdgeOrder.Prefix, seed: int = 1) -> List[CsrBatch]:
    """Consecutive update batches of `batch_size` edges (0 = one bulk batch); every batch spans the
    full vertex count (io/batching.hpp:46-66)."""
    s, d = edge_sequence(csr)
    if order == EdgeOrder.Shuffled:
        p = deterministic_shuffle(s.size, seed)
        s, d = s[p], d[p]
    if batch_size == 0:
        batch_size = s.size
    if s.size == 0:
        return [_batch_from_pairs(kind, csr.vertex_count, s, d)]
    return [_batch_from_pairs(kind, csr.vertex_count, s[b:b + batch_size], d[b:b + batch_size])
            for b in range(0, s.size, batch_size)]


# ---------------------------------------------------------------------------
# workload runner (io/workload.hpp)
# ---------------------------------------------------------------------------
class OpsMode(Enum):
    Insert = 0
    Delete = 1
    InsertThenDelete = 2
    QuerySample = 3


class Source(Enum):
    MatrixMarket = 0
    EdgeList = 1
    SynthUniform = 2
    SynthPowerLaw = 3


@dataclass
class WorkloadSpec:
    """io/workload.hpp:26-43."""
    graph_name: str = "graph"
    source: Source = Source.MatrixMarket
    input_path: str = ""
    synth_vertices: int = 0
    synth_edges: int = 0
    symmetrize: bool = False
    batch_size: int = 0          # 0 = bulk
    ops: OpsMode = OpsMode.Insert
    order: EdgeOrder = EdgeOrder.Prefix
    seed: int = 1
    block_size: int = 0          # 0 = auto (from the first batch)
    query_sample: int = 1000
    config: GraphConfig = field(default_factory=GraphConfig)


@dataclass
class PhaseRow:
    phase: str
    ms: float
    memory: dict


@dataclass
class RunReport:
    """io/workload.hpp:54-73."""
    graph_name: str = ""
    batch_size: int = 0
    vertex_count: int = 0
    edges_inserted: int = 0
    edges_deleted: int = 0
    queries_run: int = 0
    queries_hit: int = 0
    effective_block_size: int = 0
    rows: List[PhaseRow] = field(default_factory=list)
    final_stats: dict = field(default_factory=dict)

    def total_ms(self, phase: str) -> float:
        return sum(r.ms for r in self.rows if r.phase == phase)


ClockFn = Callable[[], int]   # nanoseconds


def steady_clock_ns() -> ClockFn:
    return time.perf_counter_ns


def load_source(spec: WorkloadSpec) -> Csr:
    if spec.source == Source.MatrixMarket:
        return load_matrix_market(spec.input_path, spec.symmetrize)
    if spec.source == Source.EdgeList:
        return load_edge_list(spec.input_path, spec.symmetrize)
    if spec.source == Source.SynthUniform:
        return synth_uniform(spec.synth_vertices, spec.synth_edges, spec.seed)
    if spec.source == Source.SynthPowerLaw:
        return synth_power_law(spec.synth_vertices, spec.synth_edges, spec.seed)
    raise DataError("unknown workload source")


def query_sample_pairs(csr: Csr, count: int, seed: int):
    """The query mix of io/workload.hpp:156-176: even draws sample an input edge, odd draws a
    uniform pair; one mt19937_64 stream seeded with seed ^ 0x9e3779b97f4a7c15."""
    rng = Mt19937_64(seed ^ 0x9E3779B97F4A7C15)
    qs = np.zeros(count, np.uint32)
    qd = np.zeros(count, np.uint32)
    E, V = csr.edge_count(), csr.vertex_count
    off = csr.offsets.astype(np.uint64)
    for i in range(count):
        if i % 2 == 0 and E > 0:
            e = rng() % E
            # largest v in [0, V) with offsets[v] <= e (the reference's lo/hi search)
            qs[i] = min(int(np.searchsorted(off[:V], np.uint64(e), side="right")) - 1, V - 1)
            qd[i] = csr.destinations[e]
        else:
            qd[i] = rng() % V   # (drawn first, see the module docstring)
            qs[i] = rng() % V
    return qs, qd


def run_workload(spec: WorkloadSpec, csr: Optional[Csr] = None, clock: Optional[ClockFn] = None) -> RunReport:
    """init -> insert batches -> optional delete batches -> query sample, one timed row and one
    memory snapshot per phase (io/workload.hpp:104-190).  Timing covers engine work only: parsing
    and batch construction happen before the clock starts, and every op returns after the device
    finished (the C ABI is synchronous)."""
    if csr is None:
        csr = load_source(spec)
    clock = clock or steady_clock_ns()
    report = RunReport(graph_name=spec.graph_name, batch_size=spec.batch_size, vertex_count=csr.vertex_count)
    insert_batch_size = 0 if spec.ops == OpsMode.Delete else spec.batch_size
    insert_batches = make_batches(csr, insert_batch_size, BatchKind.Insert, spec.order, spec.seed)
    block_size = spec.block_size
    if block_size == 0:
        block_size = compute_block_size(insert_batches[0]) if insert_batches[0].edge_count() > 0 else 1
    report.effective_block_size = block_size

    def timed(phase, body):
        start = clock()
        body()
        stop = clock()
        return PhaseRow(phase, (stop - start) / 1e6, {})

    box = {}
    row = timed("init", lambda: box.setdefault("g", DynamicGraph(spec.config, csr.vertex_count, block_size)))
    graph: DynamicGraph = box["g"]
    row.memory = graph.memory()
    report.rows.append(row)
    try:
        for batch in insert_batches:
            row = timed("insert", lambda: graph.insert_batch(batch))
            row.memory = graph.memory()
            report.rows.append(row)
            report.edges_inserted += batch.edge_count()
        if spec.ops in (OpsMode.Delete, OpsMode.InsertThenDelete):
            for batch in make_batches(csr, spec.batch_size, BatchKind.Delete, spec.order, spec.seed):
                row = timed("delete", lambda: graph.delete_batch(batch))
                row.memory = graph.memory()
                report.rows.append(row)
                report.edges_deleted += batch.edge_count()
        if spec.query_sample > 0 and csr.vertex_count > 0:
            qs, qd = query_sample_pairs(csr, spec.query_sample, spec.seed)
            hits = {}
            # the reference loops over query_edge; the GPU store answers the whole sample in one batched call
            row = timed("query", lambda: hits.setdefault("n", int(np.count_nonzero(graph.query_edges(qs, qd)))))
            row.memory = graph.memory()
            report.rows.append(row)
            report.queries_run = int(qs.size)
            report.queries_hit = hits["n"]
        report.final_stats = graph.stats()
    finally:
        graph.close()
    return report


def write_csv(report: RunReport) -> str:
    """One row per phase, the reference's schema (io/workload.hpp:197-208).  The byte columns are
    REAL device allocations here (dg_memory), not the reference's simulated arena accounting."""
    out = ["graph,batch_size,phase,ms,bytes_dict,bytes_sentinel,bytes_pool,bytes_total\n"]
    batch = "bulk" if report.batch_size == 0 else str(report.batch_size)
    for row in report.rows:
        m = row.memory
        out.append(f"{report.graph_name},{batch},{row.phase},{row.ms:.3f},{m['dictionary_bytes']},"
                   f"{m['sentinel_bytes']},{m['pool_bytes']},{m['total']}\n")
    return "".join(out)
