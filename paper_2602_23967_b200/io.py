"""Instance files: a binary CSR format for scale, the reference's JSON
documents and QPS text.

* ``.aqpz`` -- this package's binary format: one uncompressed NumPy ``.npz``
  holding the CSR arrays (int64 indptr/indices, float64 values) and vectors
  exactly as :class:`~.model.QpProblem` keeps them, plus a small JSON header.
  Loading is a straight read (no parsing), so C5 (5e8 nonzeros) loads at disk
  speed; the reference's JSON COO triplets (``aq/serialize.py:21-38``) cannot
  hold instances of that size.
* ``.json`` -- the reference's problem document (``aq/serialize.py:55-112``):
  COO triplets, ``null`` for infinite bounds; read and written compatibly.
* ``.qps`` / ``.mps`` -- QPS text with the reference reader's conventions
  (``aq/qps.py:1-16``): sections NAME ROWS COLUMNS RHS RANGES BOUNDS
  QUADOBJ/QMATRIX ENDATA, default bounds [0, inf), a negative UP on an
  untouched lower bound frees it, an RHS on the objective row is the negated
  objective constant, extra N rows become free rows, quadratic entries
  assign (so listing both triangles is harmless); integer markers, integer /
  semicontinuous bounds and OBJSENSE are rejected.

All of this is host-side file handling; the solve path is untouched.
"""

from __future__ import annotations

import dataclasses
import json
import os
from typing import Dict, List, Tuple

import numpy as np

from .errors import ParseError, UnsupportedSection
from .linalg import DiagonalQuad, SparseLowRankQuad, SparseMatrix, SparseQuad
from .model import Bounds, QpProblem

BINARY_VERSION = 1


# ------------------------------------------------------------------ binary (.aqpz)
def save_binary(problem: QpProblem, path) -> None:
    """Write ``problem`` as an uncompressed .npz (``.aqpz``)."""
    p = QpProblem.from_any(problem)
    q = p.quad
    arrays: Dict[str, np.ndarray] = {}

    def put_csr(tag, m: SparseMatrix):
        arrays[f"{tag}_indptr"] = np.asarray(m.indptr, dtype=np.int64)
        arrays[f"{tag}_indices"] = np.asarray(m.indices, dtype=np.int64)
        arrays[f"{tag}_data"] = np.asarray(m.data, dtype=np.float64)

    put_csr("a", p.constraint_matrix)
    if q.kind == "diagonal":
        arrays["q_values"] = np.asarray(q.values, dtype=np.float64)
    else:
        pq = q if q.kind == "sparse" else q.p
        put_csr("q", pq.upper)
        arrays["q_diag"] = np.asarray(pq.diag, dtype=np.float64)
        if q.kind == "sparse_low_rank":
            put_csr("r", q.r)
    arrays["cost"] = np.asarray(p.cost, dtype=np.float64)
    arrays["var_lower"], arrays["var_upper"] = p.var_bounds.lower, p.var_bounds.upper
    arrays["con_lower"], arrays["con_upper"] = p.con_bounds.lower, p.con_bounds.upper
    header = {"format": "aqpz", "version": BINARY_VERSION, "name": p.name, "n": p.n, "m": p.m,
              "quad": q.kind, "r_rows": q.r.rows if q.kind == "sparse_low_rank" else 0}
    arrays["header"] = np.frombuffer(json.dumps(header).encode(), dtype=np.uint8)
    path = os.fspath(path)
    with open(path, "wb") as fh:  # a file object keeps numpy from appending ".npz"
        np.savez(fh, **arrays)


def load_binary(path) -> QpProblem:
    try:
        z = np.load(os.fspath(path), allow_pickle=False)
    except (ValueError, OSError) as exc:
        raise ParseError(f"not a binary instance: {exc}") from exc
    try:
        header = json.loads(bytes(z["header"]).decode())
        if header.get("format") != "aqpz" or header.get("version") != BINARY_VERSION:
            raise ParseError(f"unsupported binary instance header {header!r}")
        n, m = int(header["n"]), int(header["m"])

        def csr(tag, rows, cols):
            return SparseMatrix(rows, cols, z[f"{tag}_indptr"], z[f"{tag}_indices"], z[f"{tag}_data"])

        kind = header["quad"]
        if kind == "diagonal":
            quad = DiagonalQuad(z["q_values"])
        elif kind == "sparse":
            quad = SparseQuad(csr("q", n, n), z["q_diag"])
        elif kind == "sparse_low_rank":
            quad = SparseLowRankQuad(SparseQuad(csr("q", n, n), z["q_diag"]), csr("r", int(header["r_rows"]), n))
        else:
            raise ParseError(f"unknown quadratic kind {kind!r}")
        return QpProblem(quad=quad, cost=z["cost"], constraint_matrix=csr("a", m, n),
                         var_bounds=Bounds(z["var_lower"], z["var_upper"]),
                         con_bounds=Bounds(z["con_lower"], z["con_upper"]), name=header.get("name", ""))
    except KeyError as exc:
        raise ParseError(f"binary instance lacks array {exc}") from exc
    finally:
        z.close()


# ------------------------------------------------------------------ reference JSON documents
def _coo_doc(mat: SparseMatrix) -> dict:
    rows = np.repeat(np.arange(mat.rows), np.diff(mat.indptr))
    return {"rows": int(mat.rows), "cols": int(mat.cols),
            "entries": [[int(i), int(j), float(v)] for i, j, v in zip(rows, mat.indices, mat.data)]}


def _csr_of_doc(doc) -> SparseMatrix:
    e = doc.get("entries", [])
    arr = np.asarray(e, dtype=np.float64).reshape(-1, 3) if e else np.zeros((0, 3))
    return SparseMatrix.from_coo(int(doc["rows"]), int(doc["cols"]), arr[:, 0].astype(np.int64),
                                 arr[:, 1].astype(np.int64), arr[:, 2])


def _nullable(v, inf):
    return [None if x == inf else float(x) for x in v]


def problem_to_dict(problem: QpProblem) -> dict:
    """The reference's problem document (``aq/serialize.py:55-80``)."""
    p = QpProblem.from_any(problem)
    q = p.quad
    if q.kind == "diagonal":
        qd = {"kind": "diagonal", "values": [float(v) for v in q.values]}
    elif q.kind == "sparse":
        qd = {"kind": "sparse", "upper": _coo_doc(q.upper)}
    else:
        qd = {"kind": "sparse_low_rank", "upper": _coo_doc(q.p.upper), "factor": _coo_doc(q.r)}
    return {"name": p.name, "quad": qd, "cost": [float(v) for v in p.cost],
            "constraint_matrix": _coo_doc(p.constraint_matrix),
            "var_lower": _nullable(p.var_bounds.lower, -np.inf), "var_upper": _nullable(p.var_bounds.upper, np.inf),
            "con_lower": _nullable(p.con_bounds.lower, -np.inf), "con_upper": _nullable(p.con_bounds.upper, np.inf)}


def problem_from_dict(doc: dict) -> QpProblem:
    """Inverse of :func:`problem_to_dict` (``aq/serialize.py:83-112``)."""

    def bounds(lo, up):
        return Bounds(np.array([-np.inf if v is None else float(v) for v in lo], dtype=np.float64),
                      np.array([np.inf if v is None else float(v) for v in up], dtype=np.float64))

    try:
        qd = doc["quad"]
        kind = qd["kind"]
        if kind == "diagonal":
            quad = DiagonalQuad(np.asarray(qd["values"], dtype=np.float64))
        elif kind == "sparse":
            quad = SparseQuad(_csr_of_doc(qd["upper"]))
        elif kind == "sparse_low_rank":
            quad = SparseLowRankQuad(SparseQuad(_csr_of_doc(qd["upper"])), _csr_of_doc(qd["factor"]))
        else:
            raise ParseError(f"unknown quadratic kind {kind!r}")
        return QpProblem(quad=quad, cost=np.asarray(doc["cost"], dtype=np.float64),
                         constraint_matrix=_csr_of_doc(doc["constraint_matrix"]),
                         var_bounds=bounds(doc["var_lower"], doc["var_upper"]),
                         con_bounds=bounds(doc["con_lower"], doc["con_upper"]), name=doc.get("name", ""))
    except (KeyError, TypeError, IndexError) as exc:
        raise ParseError(f"malformed problem document: {exc}") from exc


def dump_problem_json(problem: QpProblem, path) -> None:
    with open(path, "w") as fh:
        json.dump(problem_to_dict(problem), fh)
        fh.write("\n")


def load_problem_json(path) -> QpProblem:
    with open(path) as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise ParseError(f"invalid JSON: {exc}") from exc
    return problem_from_dict(doc)


# ------------------------------------------------------------------ QPS
@dataclasses.dataclass
class QpsDocument:
    """A parsed QPS file: the problem and its objective constant."""

    problem: QpProblem
    objective_constant: float = 0.0


_HEADERS = ("NAME", "ROWS", "COLUMNS", "RHS", "RANGES", "BOUNDS", "QUADOBJ", "QMATRIX", "OBJSENSE", "ENDATA")
_NOT_SUPPORTED_BOUNDS = ("BV", "LI", "UI", "SC")


class _QpsReader:
    """Line-by-line state machine; arrays are assembled once at the end."""

    def __init__(self, name: str):
        self.name = name
        self.section = None
        self.objective = None        # name of the first N row
        self.kind: Dict[str, str] = {}   # row name -> L/G/E/N (extra N rows are free)
        self.rows: List[str] = []        # constraint rows in file order
        self.cols: Dict[str, int] = {}   # column name -> index in first-seen order
        self.c: Dict[int, float] = {}
        self.a_r: List[str] = []
        self.a_c: List[int] = []
        self.a_v: List[float] = []
        self.rhs: Dict[str, float] = {}
        self.rng: Dict[str, float] = {}
        self.bnd: List[Tuple[str, int, float]] = []
        self.q: Dict[Tuple[int, int], float] = {}
        self.constant = 0.0

    # helpers
    def err(self, msg, line):
        return ParseError(msg, line, self.section)

    def col(self, tok):
        j = self.cols.get(tok)
        if j is None:
            j = self.cols[tok] = len(self.cols)
        return j

    def num(self, tok, line):
        try:
            return float(tok)
        except ValueError:
            raise self.err(f"bad numeric field {tok!r}", line) from None

    def known_row(self, tok, line):
        if tok not in self.kind and tok != self.objective:
            raise self.err(f"unknown row {tok!r}", line)
        return tok

    # sections
    def header(self, toks, line):
        key = toks[0].upper()
        if key not in _HEADERS:
            raise UnsupportedSection(f"section {key!r} is not supported", line)
        if key == "OBJSENSE":
            raise UnsupportedSection("OBJSENSE is not supported (minimization only)", line)
        self.section = key
        if key == "NAME" and len(toks) > 1:
            self.name = toks[1]
        return key != "ENDATA"

    def on_rows(self, t, line):
        if len(t) != 2:
            raise self.err("ROWS lines need a type and a name", line)
        typ, nm = t[0].upper(), t[1]
        if typ not in ("N", "L", "G", "E"):
            raise self.err(f"unknown row type {typ!r}", line)
        if nm in self.kind or nm == self.objective:
            raise self.err(f"duplicate row {nm!r}", line)
        if typ == "N" and self.objective is None:
            self.objective = nm
            return
        self.kind[nm] = typ
        self.rows.append(nm)

    def on_columns(self, t, line):
        if any(x.upper().strip("'") in ("MARKER", "INTORG", "INTEND") for x in t):
            raise UnsupportedSection("integer markers are not supported", line)
        if len(t) < 3 or len(t) % 2 == 0:
            raise self.err("COLUMNS lines need col then row/value pairs", line)
        j = self.col(t[0])
        for k in range(1, len(t), 2):
            v = self.num(t[k + 1], line)
            r = self.known_row(t[k], line)
            if r == self.objective:
                self.c[j] = self.c.get(j, 0.0) + v
            else:
                self.a_r.append(r)
                self.a_c.append(j)
                self.a_v.append(v)

    def on_rhs_ranges(self, t, line):
        if len(t) < 2:
            raise self.err(f"{self.section} lines need row/value pairs", line)
        pairs = t[1:] if len(t) % 2 else t  # optional leading set name
        for k in range(0, len(pairs) - 1, 2):
            v = self.num(pairs[k + 1], line)
            if self.section == "RHS" and pairs[k] == self.objective:
                self.constant = -v
                continue
            (self.rhs if self.section == "RHS" else self.rng)[self.known_row(pairs[k], line)] = v

    def on_bounds(self, t, line):
        typ = t[0].upper()
        if typ in _NOT_SUPPORTED_BOUNDS:
            raise UnsupportedSection(f"bound type {typ!r} is not supported", line)
        if typ in ("FR", "MI", "PL"):
            if len(t) < 2:
                raise self.err("bound line is too short", line)
            self.bnd.append((typ, self.col(t[2] if len(t) >= 3 else t[1]), 0.0))
        elif typ in ("UP", "LO", "FX"):
            if len(t) >= 4:
                ctok, vtok = t[2], t[3]
            elif len(t) == 3:
                ctok, vtok = t[1], t[2]
            else:
                raise self.err("bound line is too short", line)
            self.bnd.append((typ, self.col(ctok), self.num(vtok, line)))
        else:
            raise self.err(f"unknown bound type {typ!r}", line)

    def on_quad(self, t, line):
        if len(t) != 3:
            raise self.err("quadratic lines need two columns and a value", line)
        i, j = self.col(t[0]), self.col(t[1])
        self.q[(min(i, j), max(i, j))] = self.num(t[2], line)  # assign: both triangles are harmless

    def feed(self, text: str):
        handlers = {"ROWS": self.on_rows, "COLUMNS": self.on_columns, "RHS": self.on_rhs_ranges,
                    "RANGES": self.on_rhs_ranges, "BOUNDS": self.on_bounds, "QUADOBJ": self.on_quad,
                    "QMATRIX": self.on_quad}
        for line, raw in enumerate(text.splitlines(), start=1):
            s = raw.strip()
            if not s or s[0] in "*$":
                continue
            t = raw.split()
            if not raw[0].isspace():
                if not self.header(t, line):
                    break
                continue
            if self.section is None:
                raise ParseError("data line before any section header", line)
            h = handlers.get(self.section)
            if h is not None:
                h(t, line)
            elif self.section == "NAME":
                self.name = t[0]
            else:
                raise self.err(f"unexpected data in section {self.section}", line)

    def build(self) -> QpsDocument:
        if self.objective is None:
            raise ParseError("no objective (N) row found", None, "ROWS")
        n, m = len(self.cols), len(self.rows)
        cost = np.zeros(n)
        for j, v in self.c.items():
            cost[j] = v
        pos = {r: k for k, r in enumerate(self.rows)}
        lo_c, up_c = np.full(m, -np.inf), np.full(m, np.inf)
        for r, k in pos.items():
            typ, b = self.kind[r], self.rhs.get(r, 0.0)
            if typ in ("L", "E"):
                up_c[k] = b
            if typ in ("G", "E"):
                lo_c[k] = b
            if r in self.rng:
                w = self.rng[r]
                if typ == "L":
                    lo_c[k] = up_c[k] - abs(w)
                elif typ == "G":
                    up_c[k] = lo_c[k] + abs(w)
                elif typ == "E":
                    if w >= 0:
                        up_c[k] = lo_c[k] + w
                    else:
                        lo_c[k] = up_c[k] + w
        lo_v, up_v = np.zeros(n), np.full(n, np.inf)
        lower_set = np.zeros(n, dtype=bool)
        for typ, j, v in self.bnd:  # file order
            if typ == "UP":
                up_v[j] = v
                if v < 0 and not lower_set[j]:
                    lo_v[j] = -np.inf
            elif typ == "PL":
                up_v[j] = np.inf
            else:
                lower_set[j] = True
                if typ == "LO":
                    lo_v[j] = v
                elif typ == "FX":
                    lo_v[j] = up_v[j] = v
                elif typ == "MI":
                    lo_v[j] = -np.inf
                else:  # FR
                    lo_v[j], up_v[j] = -np.inf, np.inf
        a = SparseMatrix.from_coo(m, n, np.array([pos[r] for r in self.a_r], dtype=np.int64),
                                  np.array(self.a_c, dtype=np.int64), np.array(self.a_v, dtype=np.float64))
        if not self.q:
            quad = DiagonalQuad(np.zeros(n))
        elif all(i == j for i, j in self.q):
            d = np.zeros(n)
            for (i, _), v in self.q.items():
                d[i] = v
            quad = DiagonalQuad(d)
        else:
            ij = np.array(list(self.q.keys()), dtype=np.int64)
            quad = SparseQuad(SparseMatrix.from_coo(n, n, ij[:, 0], ij[:, 1], np.array(list(self.q.values()))))
        prob = QpProblem(quad=quad, cost=cost, constraint_matrix=a, var_bounds=Bounds(lo_v, up_v),
                         con_bounds=Bounds(lo_c, up_c), name=self.name)
        return QpsDocument(prob, self.constant)


def parse_qps(text: str, name: str = "") -> QpsDocument:
    """QPS text -> problem + objective constant (``aq/qps.py:43-290`` semantics)."""
    rd = _QpsReader(name)
    rd.feed(text)
    return rd.build()


def _g(v: float) -> str:
    return format(float(v), ".17g")


def write_qps(problem: QpProblem, objective_constant: float = 0.0) -> str:
    """QPS text for a diagonal or sparse problem (low-rank Q has no QPS form).

    Rows: E for equal finite bounds, L (+ RANGES) for two different finite
    bounds, L / G for one, N for none; columns X0000001..., rows R0000001...;
    values printed with 17 significant digits, so parse(write(p)) == p."""
    p = QpProblem.from_any(problem)
    if p.quad.kind not in ("diagonal", "sparse"):
        raise ValueError("QPS cannot represent low-rank quadratic operators; use JSON or .aqpz")
    n, m = p.n, p.m
    X = [f"X{i + 1:07d}" for i in range(n)]
    R = [f"R{j + 1:07d}" for j in range(m)]
    lc, uc = p.con_bounds.lower, p.con_bounds.upper
    fin_l, fin_u = np.isfinite(lc), np.isfinite(uc)
    out = [f"NAME          {p.name or 'ANONQP'}", "ROWS", " N  OBJ"]
    ranged = []
    for j in range(m):
        if fin_l[j] and fin_u[j]:
            typ = "E" if lc[j] == uc[j] else "L"
            if typ == "L":
                ranged.append(j)
        else:
            typ = "L" if fin_u[j] else ("G" if fin_l[j] else "N")
        out.append(f" {typ}  {R[j]}")
    out.append("COLUMNS")
    out += [f"    {X[i]}  OBJ  {_g(p.cost[i])}" for i in np.flatnonzero(p.cost)]
    a = p.constraint_matrix
    for j in range(m):
        for k in range(a.indptr[j], a.indptr[j + 1]):
            out.append(f"    {X[a.indices[k]]}  {R[j]}  {_g(a.data[k])}")
    out.append("RHS")
    if objective_constant != 0.0:
        out.append(f"    RHS  OBJ  {_g(-objective_constant)}")
    for j in range(m):
        v = uc[j] if fin_u[j] else (lc[j] if fin_l[j] else 0.0)
        if fin_l[j] and fin_u[j] and lc[j] == uc[j]:
            v = lc[j]
        if v != 0.0:
            out.append(f"    RHS  {R[j]}  {_g(v)}")
    if ranged:
        out.append("RANGES")
        out += [f"    RNG  {R[j]}  {_g(uc[j] - lc[j])}" for j in ranged]
    out.append("BOUNDS")
    lv, uv = p.var_bounds.lower, p.var_bounds.upper
    for i in range(n):
        fl, fu = np.isfinite(lv[i]), np.isfinite(uv[i])
        if fl and fu and lv[i] == uv[i]:
            out.append(f" FX BND  {X[i]}  {_g(lv[i])}")
        elif not fl and not fu:
            out.append(f" FR BND  {X[i]}")
        else:
            if not fl:
                out.append(f" MI BND  {X[i]}")
            elif lv[i] != 0.0:
                out.append(f" LO BND  {X[i]}  {_g(lv[i])}")
            if fu:
                out.append(f" UP BND  {X[i]}  {_g(uv[i])}")
    q = p.quad
    if q.kind == "diagonal":
        ql = [f"    {X[i]}  {X[i]}  {_g(q.values[i])}" for i in np.flatnonzero(q.values)]
    else:
        u = q.upper
        ql = [f"    {X[i]}  {X[u.indices[k]]}  {_g(u.data[k])}" for i in range(n)
              for k in range(u.indptr[i], u.indptr[i + 1])]
    if ql:
        out += ["QUADOBJ"] + ql
    out.append("ENDATA")
    return "\n".join(out) + "\n"


# ------------------------------------------------------------------ dispatch
def load_problem(path, fmt: str = None) -> QpProblem:
    """Read an instance file; the format follows the extension by default
    (``.aqpz`` binary, ``.json`` document, anything else QPS) as in the
    reference's ``aq/bench.py:53-63``."""
    path = os.fspath(path)
    if fmt is None:
        fmt = "aqpz" if path.endswith(".aqpz") else ("json" if path.endswith(".json") else "qps")
    if fmt == "aqpz":
        return load_binary(path)
    if fmt == "json":
        return load_problem_json(path)
    if fmt == "qps":
        with open(path) as fh:
            return parse_qps(fh.read(), name=os.path.basename(path)).problem
    raise ValueError(f"unknown format {fmt!r}")


def save_problem(problem: QpProblem, path, fmt: str = None) -> None:
    path = os.fspath(path)
    if fmt is None:
        fmt = "aqpz" if path.endswith(".aqpz") else ("json" if path.endswith(".json") else "qps")
    if fmt == "aqpz":
        save_binary(problem, path)
    elif fmt == "json":
        dump_problem_json(problem, path)
    elif fmt == "qps":
        with open(path, "w") as fh:
            fh.write(write_qps(problem))
    else:
        raise ValueError(f"unknown format {fmt!r}")


__all__ = ["save_binary", "load_binary", "problem_to_dict", "problem_from_dict", "dump_problem_json",
           "load_problem_json", "QpsDocument", "parse_qps", "write_qps", "load_problem", "save_problem"]
