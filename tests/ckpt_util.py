"""Test helper: read / rewrite kernelseer-checkpoint/1 files with numpy
(format: proj/docs/formats.md:53-93) so tests can perturb weights and hand the
same file to the engine and to the oracle."""
from __future__ import annotations

import numpy as np


def read(path):
    raw = open(path, "rb").read()
    sep = raw.index(b"\n\n")
    header = raw[:sep].decode().split("\n")
    payload = raw[sep + 2:]
    tensors, order, off = {}, [], 0
    for line in header:
        if line.startswith("tensor: "):
            name, shape = line[8:].rsplit(" ", 1)
            dims = [int(d) for d in shape.split("x")]
            n = int(np.prod(dims))
            tensors[name] = np.frombuffer(payload, "<f4", n, off).reshape(dims).copy()
            order.append(name)
            off += 4 * n
    return header, order, tensors


def write(path, header, order, tensors):
    with open(path, "wb") as f:
        f.write(("\n".join(header) + "\n\n").encode())
        for name in order:
            f.write(np.ascontiguousarray(tensors[name], "<f4").tobytes())


def modified(src, dst, fn):
    """Copies checkpoint src to dst after fn(tensors) edits the dict in place."""
    header, order, tensors = read(src)
    fn(tensors)
    write(dst, header, order, tensors)
    return dst
