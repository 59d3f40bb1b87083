"""Kernel tuning-parameter schemas (Table I of the paper) and the synthetic
problem-descriptor grids.

Mirrors builtin_specs() (proj/src/constraints.cpp:111-169, pinned by
proj/tests/fixtures/table1.txt) and the descriptor grids of
generate_synthetic (proj/src/data.cpp:355-359).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Tuple


@dataclass
class KernelSpec:
    name: str
    params: List[Tuple[str, List[int]]] = field(default_factory=list)

    def num_params(self) -> int:
        return len(self.params)

    def param_index(self, name: str) -> int:
        for i, (n, _) in enumerate(self.params):
            if n == name:
                return i
        return -1

    def __repr__(self) -> str:
        return f"<KernelSpec {self.name} ({len(self.params)} params)>"


def _rng(lo, hi):
    return list(range(lo, hi + 1))


def _pow2(lo, hi):
    return [1 << e for e in range(lo, hi + 1)]


BUILTIN_SPECS: Dict[str, KernelSpec] = {
    s.name: s
    for s in [
        KernelSpec("ConvAsm1x1U", [
            ("read_size", _rng(1, 4)), ("k_mult", [1, 4, 8, 16, 32]),
            ("chunks_per_wave", _rng(1, 16)), ("chunk_size", [1, 2, 4, 8, 16, 32, 64]),
            ("n_mult", _rng(1, 8)), ("c_mult", [1, 2, 4, 8, 16, 32]),
            ("waves_c_in_group", _rng(1, 8)), ("waves_k_in_group", [1, 2, 4, 8])]),
        KernelSpec("ConvOclDirectFwd1x1", [
            ("grp_tile1", _pow2(0, 4)), ("grp_tile0", _pow2(0, 8)), ("in_tile1", _pow2(0, 5)),
            ("in_tile_0", _pow2(0, 5)), ("out_pix_tile1", [0, 1]), ("out_pix_tile0", [0, 1, 2, 4]),
            ("n_out_pix_tiles", _pow2(0, 6)), ("n_in_data_tiles", _pow2(0, 11)),
            ("n_stacks", [0, 1])]),
        KernelSpec("ConvAsmBwdWrW1x1", [
            ("read_size", _rng(1, 4)), ("c_per_gpr", [1, 2, 4, 8, 16]), ("c_mult", [1, 2, 4, 8, 16]),
            ("k_per_gpr", [1, 2, 4, 8, 16]), ("k_mult", [1, 2, 4, 8, 16]),
            ("n_per_gpr", [1, 2, 4, 8, 16]), ("n_part_cnt", _rng(1, 8)),
            ("chunk_size", [1, 2, 4, 8, 16]), ("short_store", [0, 1]), ("data_prefetch", _rng(0, 4))]),
        KernelSpec("ConvAsmBwdWrW3x3", [
            ("limit_wave_cnt", _rng(0, 9)), ("reverse_inout", [0, 1]), ("chunk_size", [8, 16]),
            ("k_per_wave", [1, 2, 4, 8]), ("pipe_lines_depth", _rng(1, 16)),
            ("n_per_group", _rng(1, 8))]),
    ]
}

# generate_synthetic's descriptor grids (data.cpp:355-358); y = x = 1, or 3 for 3x3 kernels
N_GRID = [1, 2, 4, 32, 48, 64, 192, 224, 256]
CK_GRID = [16, 24, 32, 192, 256, 320, 768, 896, 1024]
HW_GRID = [7, 10, 14, 48, 56, 64, 192, 224]
FIELDS = ["n", "c", "h", "w", "k", "y", "x"]


def input_grids(kernel: str):
    f = 3 if "3x3" in kernel else 1
    return [N_GRID, CK_GRID, HW_GRID, HW_GRID, CK_GRID, [f], [f]]


def search_space_size(spec: KernelSpec) -> int:
    n = 1
    for _, v in spec.params:
        n *= len(v)
    return n
