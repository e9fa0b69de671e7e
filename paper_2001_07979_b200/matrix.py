"""Parity-check matrices H_1..H_u and the stacked edge layout the device decodes on.

Host-side data formats on the drop-in boundary.  The decoder accepts either
these classes or the reference package's own (``mmrecon.matrix``): anything
with ``n``, ``m``, ``chk_ptr``, ``chk_var`` (a matrix) or ``matrices`` (an
ensemble) is understood, so a caller that builds its PEG ensemble with the
reference keeps doing so.

Reference: ``ParityCheckMatrix`` / ``MatrixEnsemble`` (pkg/src/mmrecon/matrix.py:71-212),
the stacked layout of ``DecoderWorkspace`` (pkg/src/mmrecon/decoder.py:80-122).
PEG construction (matrix.py:215-260) is restated exactly in
the native library (``peg_construct`` / ``build_ensemble``, csrc/peg.cpp); the
benchmark ensembles also ship as compact caches produced by the reference's
``build_ensemble`` (``tests/golden/make_ensembles.py``).
"""

from __future__ import annotations

import hashlib
import io
from dataclasses import dataclass
from pathlib import Path

import numpy as np

__all__ = [
    "ParityCheckMatrix",
    "MatrixEnsemble",
    "StackedLayout",
    "stacked_layout",
    "save_ensemble",
    "load_ensemble",
    "code_rate",
    "random_regular_matrix",
    "random_regular_ensemble",
    "peg_construct",
    "build_ensemble",
]

ENSEMBLE_CACHE_VERSION = 1


class ParityCheckMatrix:
    """GF(2) Tanner graph in dual CSR form (check side and variable side).

    Same invariants as the reference (matrix.py:86-115): 0 < m < n, rows
    sorted, no parallel edges, no empty column.  Arrays are read-only.
    """

    __slots__ = ("n", "m", "chk_ptr", "chk_var", "var_ptr", "var_chk", "_hash")

    def __init__(self, n, m, chk_ptr, chk_var, var_ptr, var_chk):
        self.n = int(n)
        self.m = int(m)
        self.chk_ptr = np.asarray(chk_ptr, dtype=np.int64)
        self.chk_var = np.asarray(chk_var, dtype=np.int32)
        self.var_ptr = np.asarray(var_ptr, dtype=np.int64)
        self.var_chk = np.asarray(var_chk, dtype=np.int32)
        for a in (self.chk_ptr, self.chk_var, self.var_ptr, self.var_chk):
            a.setflags(write=False)
        self._hash = None

    @classmethod
    def from_check_adjacency(cls, n: int, m: int, rows) -> "ParityCheckMatrix":
        if not 0 < m < n:
            raise ValueError(f"need 0 < m < n, got m={m}, n={n}")
        if len(rows) != m:
            raise ValueError(f"{len(rows)} adjacency rows for m={m} checks")
        sorted_rows = [np.sort(np.asarray(r, dtype=np.int64)) for r in rows]
        deg = np.fromiter((r.size for r in sorted_rows), dtype=np.int64, count=m)
        chk_ptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        chk_var = (np.concatenate(sorted_rows) if m else np.zeros(0)).astype(np.int64)
        for j, r in enumerate(sorted_rows):
            if r.size and (r[0] < 0 or r[-1] >= n):
                raise ValueError(f"check {j}: variable index out of range [0, {n})")
            if r.size > 1 and np.any(r[1:] == r[:-1]):
                raise ValueError(f"check {j}: parallel edge")
        return cls._from_csr(n, m, chk_ptr, chk_var.astype(np.int32))

    @classmethod
    def _from_csr(cls, n, m, chk_ptr, chk_var):
        col_deg = np.bincount(chk_var, minlength=n)
        if np.any(col_deg == 0):
            raise ValueError(f"variable {int(np.argmin(col_deg))} has degree 0")
        order = np.argsort(chk_var, kind="stable")
        var_ptr = np.concatenate([[0], np.cumsum(col_deg)]).astype(np.int64)
        row_of_edge = np.repeat(np.arange(m, dtype=np.int32), np.diff(chk_ptr))
        return cls(n, m, chk_ptr, chk_var, var_ptr, row_of_edge[order])

    @property
    def edge_count(self) -> int:
        return int(self.chk_var.shape[0])

    def row_adj(self, j: int) -> np.ndarray:
        return self.chk_var[self.chk_ptr[j]:self.chk_ptr[j + 1]]

    def col_adj(self, i: int) -> np.ndarray:
        return self.var_chk[self.var_ptr[i]:self.var_ptr[i + 1]]

    def row_degrees(self) -> np.ndarray:
        return np.diff(self.chk_ptr)

    def column_degrees(self) -> np.ndarray:
        return np.diff(self.var_ptr)

    def to_dense(self) -> np.ndarray:
        h = np.zeros((self.m, self.n), dtype=np.uint8)
        rows = np.repeat(np.arange(self.m), np.diff(self.chk_ptr))
        h[rows, self.chk_var] = 1
        return h

    def content_hash(self) -> str:
        """SHA-256 over (n, m, chk_ptr, chk_var); equals the reference's
        ``ParityCheckMatrix.content_hash`` (matrix.py:148-154) for the same graph.
        Memoised: the arrays are read-only."""
        if self._hash is None:
            h = hashlib.sha256()
            h.update(np.array([self.n, self.m], dtype="<i8").tobytes())
            h.update(self.chk_ptr.astype("<i8").tobytes())
            h.update(self.chk_var.astype("<i4").tobytes())
            self._hash = h.hexdigest()
        return self._hash

    def __eq__(self, other):
        if not hasattr(other, "chk_var"):
            return NotImplemented
        return (self.n == other.n and self.m == other.m
                and np.array_equal(self.chk_ptr, other.chk_ptr)
                and np.array_equal(self.chk_var, other.chk_var))

    def __hash__(self):
        return hash(self.content_hash())

    def __repr__(self):
        return f"ParityCheckMatrix(n={self.n}, m={self.m}, edges={self.edge_count})"


@dataclass(frozen=True)
class MatrixEnsemble:
    """u matrices over one variable set; members share (n, m) and differ."""

    matrices: tuple

    def __post_init__(self):
        if len(self.matrices) < 1:
            raise ValueError("ensemble needs at least one matrix")
        n, m = self.matrices[0].n, self.matrices[0].m
        for k, h in enumerate(self.matrices):
            if (h.n, h.m) != (n, m):
                raise ValueError(f"matrix {k} has shape ({h.m}, {h.n}), expected ({m}, {n})")
        for a in range(len(self.matrices)):
            for b in range(a + 1, len(self.matrices)):
                if self.matrices[a] == self.matrices[b]:
                    raise ValueError(f"matrices {a} and {b} have identical edge sets")

    @property
    def u(self) -> int:
        return len(self.matrices)

    @property
    def n(self) -> int:
        return self.matrices[0].n

    @property
    def m(self) -> int:
        return self.matrices[0].m

    def prefix(self, u: int) -> "MatrixEnsemble":
        if not 1 <= u <= self.u:
            raise ValueError(f"u={u} outside [1, {self.u}]")
        return MatrixEnsemble(tuple(self.matrices[:u]))

    def content_hashes(self) -> list:
        return [h.content_hash() for h in self.matrices]


def peg_construct(n: int, m: int, column_degree=3, seed: int = 0, device: int | None = None) -> ParityCheckMatrix:
    """Progressive-edge-growth matrix, identical to the reference's
    ``matrix.peg_construct(n, m, DegreeProfile, seed)`` (matrix.py:215-234)
    for the same seed: ``mbp_peg_build`` in the native library restates
    ``_kernels.peg_build`` (BFS order, candidate scan, xorshift64* ties).
    ``column_degree``: an int (regular) or n per-column degrees (>= 2, as
    DegreeProfile requires).  Host code is sequential: seconds at n = 2^16,
    hours at 2^20 (the reference's cost grows the same way, ~n*m).
    ``device``: run each edge's BFS on that GPU (mbp_peg_build_device, the
    same matrix; the practical route at n = 2^20)."""
    import ctypes as C

    from . import _native as N

    if not 0 < m < n:
        raise ValueError(f"need 0 < m < n, got m={m}, n={n}")
    if np.ndim(column_degree) == 0:
        if int(column_degree) < 2:
            raise ValueError(f"column degree must be >= 2, got {column_degree}")
        deg = np.full(n, int(column_degree), dtype=np.int32)
    else:
        deg = np.ascontiguousarray(column_degree, dtype=np.int32)
        if deg.shape != (n,):
            raise ValueError(f"profile lists {deg.size} degrees for n={n} columns")
        if np.any(deg < 2):
            raise ValueError("all column degrees must be >= 2")
    if int(deg.max()) > m:
        raise ValueError(f"column degree {int(deg.max())} exceeds m={m}: parallel edges would be forced")
    E = int(deg.sum())
    chk_ptr = np.zeros(m + 1, dtype=np.int64)
    chk_var = np.zeros(E, dtype=np.int32)
    if device is None:
        N.call("mbp_peg_build", int(n), int(m), deg.ctypes.data, C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF),
               chk_ptr.ctypes.data, chk_var.ctypes.data)
    else:
        N.call("mbp_peg_build_device", int(n), int(m), deg.ctypes.data,
               C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), chk_ptr.ctypes.data, chk_var.ctypes.data, int(device))
    return ParityCheckMatrix._from_csr(n, m, chk_ptr, chk_var)


def peg_device_stage(n: int, m: int, column_degree, seed: int, state: int, v_begin: int, v_end: int,
                     vn_adj: np.ndarray, device: int = 0) -> int:
    """One stage of the device PEG (mbp_peg_build_device_range): variables
    [v_begin, v_end) on top of ``vn_adj`` (int32 [n, 4], -1 = no edge; updated
    in place).  Returns the tie-break stream state at v_end (pass it to the
    next stage); ``state`` is ignored when v_begin == 0."""
    import ctypes as C

    from . import _native as N

    deg = (np.full(n, int(column_degree), dtype=np.int32) if np.ndim(column_degree) == 0
           else np.ascontiguousarray(column_degree, dtype=np.int32))
    if vn_adj.dtype != np.int32 or vn_adj.shape != (n, 4) or not vn_adj.flags.c_contiguous:
        raise ValueError("vn_adj must be a contiguous int32 array of shape (n, 4)")
    st = C.c_uint64(int(state) & 0xFFFFFFFFFFFFFFFF)
    N.call("mbp_peg_build_device_range", int(n), int(m), deg.ctypes.data, C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF),
           C.byref(st), int(v_begin), int(v_end), vn_adj.ctypes.data, int(device))
    return int(st.value)


def matrix_from_variable_rows(n: int, m: int, vn_adj: np.ndarray) -> ParityCheckMatrix:
    """The PEG matrix from per-variable check lists (check rows in ascending
    variable order, as the construction attaches them)."""
    v, k = np.nonzero(vn_adj >= 0)
    c = vn_adj[v, k].astype(np.int64)
    order = np.lexsort((v, c))
    chk_ptr = np.concatenate([[0], np.cumsum(np.bincount(c, minlength=m))]).astype(np.int64)
    return ParityCheckMatrix._from_csr(n, m, chk_ptr, v[order].astype(np.int32))


def build_ensemble(n: int, m: int, column_degree=3, u: int = 1, base_seed: int = 0,
                   workers: int | None = None, device: int | None = None) -> "MatrixEnsemble":
    """u PEG matrices from seeds base_seed..base_seed+u-1, as the reference's
    ``build_ensemble`` (matrix.py:237-256); members build in parallel
    threads (the native call releases the GIL)."""
    if u < 1:
        raise ValueError(f"u must be >= 1, got {u}")
    seeds = [base_seed + k for k in range(u)]
    if u == 1 or (workers is not None and workers <= 1):
        mats = [peg_construct(n, m, column_degree, s, device) for s in seeds]
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers or min(u, 4)) as pool:
            mats = list(pool.map(lambda s: peg_construct(n, m, column_degree, s, device), seeds))
    return MatrixEnsemble(tuple(mats))


def random_regular_matrix(n: int, m: int, dv: int = 3, seed: int = 0) -> ParityCheckMatrix:
    """A random (dv, dv*n/m)-regular Tanner graph (configuration model with
    parallel edges swapped out) -- a SYNTHETIC stand-in where the reference's
    PEG construction is out of reach (n = 2^20: ~7 h per matrix in the
    reference).  The decoder does not care how
    a graph was built; parity against the oracle holds for any graph."""
    E = n * dv
    if E % m:
        raise ValueError(f"n*dv = {E} not divisible by m = {m}")
    dc = E // m
    rng = np.random.default_rng(seed)
    var_of_socket = np.repeat(np.arange(n, dtype=np.int64), dv)
    perm = rng.permutation(E)
    chk_of_socket = perm // dc            # check socket slot -> check id
    # parallel edges: swap the variable of a duplicated (check, var) pair with
    # a random socket until none remain
    for _ in range(100):
        key = chk_of_socket * n + var_of_socket
        order = np.argsort(key, kind="stable")
        dup = order[1:][key[order[1:]] == key[order[:-1]]]
        if dup.size == 0:
            break
        other = rng.integers(0, E, size=dup.size)
        var_of_socket[dup], var_of_socket[other] = var_of_socket[other], var_of_socket[dup].copy()
    else:
        raise RuntimeError("could not remove parallel edges")
    order = np.lexsort((var_of_socket, chk_of_socket))
    chk_ptr = np.arange(0, E + 1, dc, dtype=np.int64)
    return ParityCheckMatrix._from_csr(n, m, chk_ptr, var_of_socket[order].astype(np.int32))


def random_regular_ensemble(n: int, m: int, u: int, dv: int = 3, seed: int = 0) -> "MatrixEnsemble":
    """u synthetic random regular matrices with seeds seed..seed+u-1."""
    return MatrixEnsemble(tuple(random_regular_matrix(n, m, dv, seed + l) for l in range(u)))


def code_rate(matrix) -> float:
    return 1.0 - matrix.m / matrix.n


# ---------------------------------------------------------------------------
# stacked layout (the graph the device decodes)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class StackedLayout:
    """Vertically stacked (u*m) x n graph, edges numbered check-major with
    matrix 0 first -- the numbering of decoder.py:94-111, so joint decoding
    over the ensemble is decoding of the stacked matrix.

    ``var_edge`` lists each variable's incident edge ids ascending (a stable
    argsort of ``chk_var``), the summation order of the reference's
    posterior (_kernels.py:293-301)."""

    n: int
    m: int
    u: int
    edge_off: np.ndarray   # int64[u+1]
    chk_ptr: np.ndarray    # int64[u*m+1]
    chk_var: np.ndarray    # int32[E]
    var_ptr: np.ndarray    # int64[n+1]
    var_edge: np.ndarray   # int64[E]

    @property
    def edges(self) -> int:
        return int(self.edge_off[-1])

    @property
    def max_row_degree(self) -> int:
        return int(np.diff(self.chk_ptr).max()) if self.u * self.m else 0

    @property
    def max_col_degree(self) -> int:
        return int(np.diff(self.var_ptr).max())


def _matrices_of(ensemble_or_matrix):
    if hasattr(ensemble_or_matrix, "matrices"):
        return tuple(ensemble_or_matrix.matrices)
    return (ensemble_or_matrix,)


_LAYOUTS: dict = {}


def stacked_layout(ensemble) -> StackedLayout:
    """The stacked layout of an ensemble (immutable; memoised by the
    matrices' content hashes, so a layout is built once per matrix set)."""
    mats = _matrices_of(ensemble)
    key = tuple(h.content_hash() for h in mats)
    lay = _LAYOUTS.get(key)
    if lay is None:
        lay = _build_stacked_layout(mats)
        if len(_LAYOUTS) >= 8:
            _LAYOUTS.pop(next(iter(_LAYOUTS)))
        _LAYOUTS[key] = lay
    return lay


def _build_stacked_layout(mats) -> StackedLayout:
    n, m, u = mats[0].n, mats[0].m, len(mats)
    counts = [int(np.asarray(h.chk_var).shape[0]) for h in mats]
    edge_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    chk_ptr = np.zeros(u * m + 1, dtype=np.int64)
    chk_var = np.empty(int(edge_off[-1]), dtype=np.int32)
    for l, h in enumerate(mats):
        cp = np.asarray(h.chk_ptr, dtype=np.int64)
        chk_ptr[l * m + 1:(l + 1) * m + 1] = edge_off[l] + cp[1:]
        chk_var[edge_off[l]:edge_off[l + 1]] = np.asarray(h.chk_var, dtype=np.int32)
    order = np.argsort(chk_var, kind="stable").astype(np.int64)
    col_deg = np.bincount(chk_var, minlength=n)
    var_ptr = np.concatenate([[0], np.cumsum(col_deg)]).astype(np.int64)
    for a in (edge_off, chk_ptr, chk_var, var_ptr, order):
        a.setflags(write=False)
    return StackedLayout(n, m, u, edge_off, chk_ptr, chk_var, var_ptr, order)


# ---------------------------------------------------------------------------
# compact ensemble cache (versioned; SPEC.md "compact binary cache format")
# ---------------------------------------------------------------------------

def save_ensemble(ensemble, path, seeds=None, note: str = "") -> None:
    """Write an ensemble as row degrees + per-row delta-coded column indices.

    Deltas between sorted neighbours fit uint16 for n <= 65536 and uint32
    beyond; the npz is zlib-compressed.  Content hashes are stored and
    re-checked on load."""
    mats = _matrices_of(ensemble)
    n, m = mats[0].n, mats[0].m
    dt = np.uint16 if n <= 65536 else np.uint32
    arrays = {
        "version": np.array(ENSEMBLE_CACHE_VERSION),
        "n": np.array(n), "m": np.array(m), "u": np.array(len(mats)),
        "seeds": np.array(seeds if seeds is not None else [-1] * len(mats), dtype=np.int64),
        "note": np.array(note),
    }
    for l, h in enumerate(mats):
        cp = np.asarray(h.chk_ptr, dtype=np.int64)
        cv = np.asarray(h.chk_var, dtype=np.int64)
        deg = np.diff(cp)
        delta = cv.copy()
        first = np.zeros(cv.shape[0], dtype=bool)
        first[cp[:-1][deg > 0]] = True
        delta[~first] = cv[~first] - cv[np.flatnonzero(~first) - 1]
        arrays[f"rowdeg{l}"] = deg.astype(np.uint16 if deg.max() < 65536 else np.uint32)
        arrays[f"delta{l}"] = delta.astype(dt)
        arrays[f"hash{l}"] = np.array(ParityCheckMatrix._from_csr(n, m, cp, cv.astype(np.int32)).content_hash()
                                      if not hasattr(h, "content_hash") else h.content_hash())
    buf = io.BytesIO()
    np.savez_compressed(buf, **arrays)
    Path(path).write_bytes(buf.getvalue())


def load_ensemble(path, verify: bool = True) -> MatrixEnsemble:
    with np.load(path) as z:
        if int(z["version"]) != ENSEMBLE_CACHE_VERSION:
            raise ValueError(f"unsupported ensemble cache version {int(z['version'])}")
        n, m, u = int(z["n"]), int(z["m"]), int(z["u"])
        mats = []
        for l in range(u):
            deg = z[f"rowdeg{l}"].astype(np.int64)
            delta = z[f"delta{l}"].astype(np.int64)
            chk_ptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
            # undo the per-row delta code: cumulative sum restarted at each row start
            csum = np.cumsum(delta)
            row_base = np.repeat(csum[chk_ptr[:-1][deg > 0]] - delta[chk_ptr[:-1][deg > 0]], deg[deg > 0])
            chk_var = (csum - row_base).astype(np.int32)
            h = ParityCheckMatrix._from_csr(n, m, chk_ptr, chk_var)
            if verify and h.content_hash() != str(z[f"hash{l}"]):
                raise ValueError(f"{path}: matrix {l} content hash mismatch")
            mats.append(h)
    return MatrixEnsemble(tuple(mats))
