"""paper_1111_6900_b200 — B200-native GF(2^e) bitsliced-Karatsuba matrix multiply(-accumulate).

A drop-in for the hot path of the reference package ``gf2elin`` (M4RIE, arxiv 1111.6900):
the packed (mzed) and bitsliced (mzd_slice) matrix types, slice/cling, mul/addmul, with the
same names and semantics, computed by hand-written sm_100a CUDA in libgf2e_b200.so
(C ABI: include/gf2e_b200.h).  See DESIGN.md.
"""

from . import _lib
from ._device import release_workspace
from .gf2e import DEFAULT_POLYS, FieldCtx, field_new, is_irreducible, is_primitive
from .mat_gf2 import BitMatrix, RowOpCounters, addmul as gf2_addmul, mul, mzd_addmul, mzd_mul, words_for
from .mat_packed import PackedMatrix, pack_width
from .mat_sliced import SlicedMatrix, cling, mul_by_x, mzed_cling, mzed_slice, slice_packed
from .ple_echelon import (
    PermVector,
    PleFactors,
    SingularMatrixError,
    apply_perm_cols,
    apply_perm_rows,
    col_swap,
    echelonize,
    echelonize_sliced,
    ple,
    ple_reconstruct,
    ple_sliced,
    ple_unpack,
    trsm_lower_left,
    trsm_lower_left_unit,
    trsm_sliced,
    trsm_upper_left,
)
from .matfile import load_matrix, parse as parse_matrix, save_matrix, serialize as serialize_matrix
from .newton_john import NJTable, cubic_mul, make_table, nj_gauss, nj_mul, nj_ple, nj_trsm_upper_left
from .poly_mul import (
    MulCounters,
    Schedule,
    addmul,
    addmul_packed,
    count_products,
    karatsuba_mul,
    karatsuba_mul_packed,
    karatsuba_mul_packed_host,
    mzed_mul_host,
    mzd_slice_addmul,
    mzd_slice_mul,
    mzed_addmul,
    mzed_mul,
    reduce_mod_f,
    schedule,
)

__all__ = [
    "release_workspace",
    "DEFAULT_POLYS", "FieldCtx", "field_new", "is_irreducible", "is_primitive",
    "BitMatrix", "RowOpCounters", "mul", "gf2_addmul", "mzd_mul", "mzd_addmul", "words_for",
    "PackedMatrix", "pack_width",
    "SlicedMatrix", "slice_packed", "cling", "mzed_slice", "mzed_cling", "mul_by_x",
    "SingularMatrixError", "trsm_upper_left", "trsm_lower_left", "trsm_lower_left_unit", "trsm_sliced",
    "PermVector", "PleFactors", "apply_perm_rows", "apply_perm_cols", "col_swap", "ple", "ple_sliced", "ple_unpack",
    "ple_reconstruct", "echelonize", "echelonize_sliced",
    "load_matrix", "save_matrix", "parse_matrix", "serialize_matrix",
    "NJTable", "make_table", "cubic_mul", "nj_mul", "nj_gauss", "nj_ple", "nj_trsm_upper_left",
    "MulCounters", "Schedule", "schedule", "karatsuba_mul", "karatsuba_mul_packed", "karatsuba_mul_packed_host", "mzed_mul_host", "addmul", "addmul_packed",
    "reduce_mod_f", "count_products", "mzd_slice_mul", "mzd_slice_addmul", "mzed_mul", "mzed_addmul",
]

LIB_PATH = _lib.LIB_PATH
