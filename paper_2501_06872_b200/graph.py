"""CSR/CSC container with the reference's array contract.

Restates ``potra.graph.CsrGraph`` (pkg/src/potra/graph.py:39-122) and the
helpers the transposition path needs (``edge_id_dtype`` graph.py:34-36,
``lists_are_sorted`` graph.py:309-317) so the package is usable without the
reference installed.  ``transpose_gpu`` accepts either this class or the
reference's own ``CsrGraph`` (duck-typed on the same fields) and returns an
instance of the input's class, so ``out.graph == potra.transpose_oracle(g)``
works unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["CsrGraph", "edge_id_dtype", "lists_are_sorted", "flip_orientation"]


def edge_id_dtype(num_vertices: int) -> np.dtype:
    """32-bit IDs up to 2^32 vertices, else 64-bit (graph.py:34-36)."""
    return np.dtype(np.uint32) if num_vertices <= 2**32 else np.dtype(np.uint64)


def flip_orientation(orientation: str) -> str:
    """CSR <-> CSC (baselines.py:56-57)."""
    return "CSC" if orientation == "CSR" else "CSR"


@dataclass(eq=False)
class CsrGraph:
    """Directed graph in compressed sparse row/column layout (graph.py:39-92).

    ``offsets`` is uint64[num_vertices+1] with offsets[0] == 0 and
    offsets[-1] == num_edges; ``edges`` holds the stored endpoint of each edge.
    """

    num_vertices: int
    num_edges: int
    offsets: np.ndarray
    edges: np.ndarray
    orientation: str = "CSR"

    def __post_init__(self):
        self.validate()

    def validate(self):  # graph.py:59-80
        if self.num_vertices < 0 or self.num_edges < 0:
            raise ValueError("vertex and edge counts must be non-negative")
        if self.orientation not in ("CSR", "CSC"):
            raise ValueError(f"orientation must be CSR or CSC, got {self.orientation!r}")
        if self.offsets.dtype != np.uint64:
            raise ValueError("offsets must be uint64")
        if self.offsets.shape != (self.num_vertices + 1,):
            raise ValueError(
                f"offsets must have exactly {self.num_vertices + 1} entries, "
                f"got {self.offsets.shape[0]}"
            )
        if self.edges.shape != (self.num_edges,):
            raise ValueError("edges length must equal num_edges")
        if self.offsets[0] != 0:
            raise ValueError("offsets[0] must be 0")
        if int(self.offsets[-1]) != self.num_edges:
            raise ValueError("offsets[-1] must equal num_edges")
        if self.num_vertices and np.any(np.diff(self.offsets.view(np.int64)) < 0):
            raise ValueError("non-monotone offsets")
        if self.num_edges and int(self.edges.max()) >= self.num_vertices:
            raise ValueError("edge ID >= num_vertices")

    def __eq__(self, other):  # graph.py:82-92 (dtype + array equality)
        if not hasattr(other, "offsets") or not hasattr(other, "edges"):
            return NotImplemented
        return (
            self.num_vertices == other.num_vertices
            and self.num_edges == other.num_edges
            and self.orientation == other.orientation
            and self.edges.dtype == other.edges.dtype
            and np.array_equal(self.offsets, other.offsets)
            and np.array_equal(self.edges, other.edges)
        )

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets.view(np.int64))

    def neighbors(self, v: int) -> np.ndarray:
        return self.edges[int(self.offsets[v]) : int(self.offsets[v + 1])]

    def nbytes(self) -> int:
        return self.offsets.nbytes + self.edges.nbytes

    @classmethod
    def from_edge_pairs(cls, src, dst, num_vertices, orientation="CSR") -> "CsrGraph":
        """Pairs sorted by (owner, endpoint), duplicates kept (graph.py:104-122)."""
        src = np.asarray(src)
        dst = np.asarray(dst)
        if src.shape != dst.shape:
            raise ValueError("src and dst must have equal length")
        dt = edge_id_dtype(num_vertices)
        order = np.lexsort((dst, src))
        edges = dst[order].astype(dt, copy=False)
        counts = np.bincount(src.astype(np.int64, copy=False), minlength=num_vertices)
        offsets = np.zeros(num_vertices + 1, dtype=np.uint64)
        np.cumsum(counts, out=offsets[1:])
        return cls(num_vertices, int(src.shape[0]), offsets, np.ascontiguousarray(edges), orientation)


def lists_are_sorted(g) -> bool:
    """True when every neighbour list is non-decreasing (graph.py:309-317)."""
    if g.num_edges < 2:
        return True
    nondec = np.diff(g.edges.astype(np.int64)) >= 0
    starts = g.offsets[1:-1].view(np.int64)
    starts = starts[(starts > 0) & (starts < g.num_edges)]
    nondec[starts - 1] = True
    return bool(nondec.all())
