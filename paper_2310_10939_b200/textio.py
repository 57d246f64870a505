"""Text file formats of the reference, so runs of this package drop into the same tooling:
edge lists (specluster/graph.py:287-361), label files (:364-387) and embedding files
(specluster/spectral.py:130-176), plus the SBM metadata record (generate.py:96-109).
Formats, header lines and error behaviour follow the reference; the one-vector embedding
names its own generator in the header (``GENERATOR_NAME``)."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import GraphFormatError
from .graph import Graph, from_edges

# the one-vector start vector is Philox4x64 Irwin-Hall, not the reference's PCG64 ziggurat
GENERATOR_NAME = "philox4x64-irwin-hall"
_EMBEDDING_MAGIC = "#specluster-embedding"


@dataclass
class GraphLoadResult:
    graph: Graph
    id_map: list[str] | None  # id_map[new_id] = original token; None for dense int ids
    dropped: list[int]


def load_edge_list(path, *, allow_self_loops: bool = False,
                   drop_isolated: bool = False) -> GraphLoadResult:
    """``u<TAB>v[<TAB>w]`` lines, ``#`` comments; integer ids are used as vertex ids
    (n = max id + 1), any other token set is mapped to dense ids in first-seen order."""
    raw: list[tuple[str, str, float]] = []
    int_ids = True
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) not in (2, 3):
                raise GraphFormatError(
                    f"{path}:{lineno}: expected 'u<TAB>v[<TAB>w]', got {len(parts)} fields")
            try:
                w = float(parts[2]) if len(parts) == 3 else 1.0
            except ValueError:
                raise GraphFormatError(f"{path}:{lineno}: bad weight {parts[2]!r}") from None
            if not np.isfinite(w) or w <= 0:
                raise GraphFormatError(f"{path}:{lineno}: weight must be positive, got {w}")
            raw.append((parts[0], parts[1], w))
            if int_ids:
                try:
                    int_ids = int(parts[0]) >= 0 and int(parts[1]) >= 0
                except ValueError:
                    int_ids = False
    if not raw:
        raise GraphFormatError(f"{path}: no edges found")
    ws = [w for _, _, w in raw]
    id_map = None
    if int_ids:
        us = [int(a) for a, _, _ in raw]
        vs = [int(b) for _, b, _ in raw]
        n = max(max(us), max(vs)) + 1
    else:
        index: dict[str, int] = {}
        for a, b, _ in raw:
            index.setdefault(a, len(index))
            index.setdefault(b, len(index))
        us = [index[a] for a, _, _ in raw]
        vs = [index[b] for _, b, _ in raw]
        n = len(index)
        id_map = list(index)
    g, dropped = from_edges(n, us, vs, ws, allow_self_loops=allow_self_loops,
                            drop_isolated=drop_isolated)
    if dropped and id_map is not None:
        gone = set(dropped)
        id_map = [tok for i, tok in enumerate(id_map) if i not in gone]
    return GraphLoadResult(graph=g, id_map=id_map, dropped=list(dropped))


def save_edge_list(g: Graph, path, header_comments: Sequence[str] = ()) -> None:
    """Upper triangle (u < v), tab separated, weights at 17 significant digits."""
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_offsets))
    col = np.asarray(g.col_indices, dtype=np.int64)
    w = np.ones(col.size) if g.weights is None else np.asarray(g.weights)
    up = src < col
    with open(path, "w", encoding="utf-8") as fh:
        for c in header_comments:
            fh.write(f"# {c}\n")
        fh.writelines(f"{a}\t{b}\t{x:.17g}\n" for a, b, x in zip(src[up], col[up], w[up]))


def load_labels(path, expected_n: int | None = None) -> np.ndarray:
    out: list[int] = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            try:
                out.append(int(line))
            except ValueError:
                raise GraphFormatError(f"{path}:{lineno}: bad label {line!r}") from None
    if expected_n is not None and len(out) != expected_n:
        raise GraphFormatError(
            f"{path}: found {len(out)} labels but the graph has {expected_n} vertices")
    return np.asarray(out, dtype=np.int64)


def save_labels(labels, path, header_comments: Sequence[str] = ()) -> None:
    lab = np.asarray(labels, dtype=np.int64)
    with open(path, "w", encoding="utf-8") as fh:
        for c in header_comments:
            fh.write(f"# {c}\n")
        fh.write("".join(f"{v}\n" for v in lab.tolist()))


def save_embedding(data: np.ndarray, path, *, scaled: bool, seed: int,
                   generator: str | None = None) -> None:
    """Header + one comma-separated row per vertex at 17 significant digits."""
    d = np.asarray(data, dtype=np.float64)
    if d.ndim == 1:
        d = d[:, None]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"{_EMBEDDING_MAGIC} n={d.shape[0]} l={d.shape[1]} "
                 f"scaled={1 if scaled else 0} seed={seed}\n")
        fh.write(f"# generator={generator or GENERATOR_NAME} numpy={np.__version__}\n")
        if d.shape[1] == 1:
            fh.write("".join(f"{v:.17g}\n" for v in d[:, 0].tolist()))
        else:
            for row in d.tolist():
                fh.write(",".join(f"{v:.17g}" for v in row) + "\n")


def load_embedding(path) -> tuple[np.ndarray, bool, int]:
    """-> (data (n, l), scaled, seed)."""
    with open(path, "r", encoding="utf-8") as fh:
        header = fh.readline().strip()
        if not header.startswith(_EMBEDDING_MAGIC):
            raise GraphFormatError(f"{path}:1: missing '{_EMBEDDING_MAGIC}' header")
        try:
            fields = dict(tok.split("=", 1) for tok in header.split()[1:])
            n, l = int(fields["n"]), int(fields["l"])
            scaled, seed = fields["scaled"] == "1", int(fields["seed"])
        except (KeyError, ValueError):
            raise GraphFormatError(f"{path}:1: malformed header {header!r}") from None
        rows = []
        for lineno, line in enumerate(fh, start=2):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            try:
                rows.append([float(v) for v in line.split(",")])
            except ValueError:
                raise GraphFormatError(f"{path}:{lineno}: bad row") from None
    data = np.asarray(rows, dtype=np.float64)
    if data.shape != (n, l):
        raise GraphFormatError(f"{path}: header promises {n}x{l} but file holds "
                               f"{data.shape[0]}x{data.shape[1] if data.ndim == 2 else 1}")
    return data, scaled, seed


def sbm_metadata_record(sample, generator: str) -> dict:
    p = sample.params
    return {"type": "sbm", "n": p.n, "k": p.k, "p": p.p, "q": p.q, "seed": p.seed,
            "generator": generator, "n_after_drop": sample.graph.n,
            "num_dropped": len(sample.dropped), "dropped": [int(v) for v in sample.dropped],
            "edges": sample.graph.nnz // 2}
