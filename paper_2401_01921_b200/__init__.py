"""paper_2401_01921_b200 -- a B200-native engine for the tensor-operation hot path
of the Cytnx paper (arxiv 2401.01921), behind the reference ``tnkit`` API.

Hot path (BASELINE.json north_star):
  * dense permute materialisation  -> ``tnb_permute``          (smem-tiled, 16-B lanes)
  * dense Contract / Network        -> ``tnb_contract_dense``   (FP64 DMMA, permute fused
                                                                into the operand gather)
  * U(1)/Z_n block-sparse contract -> ``tnb_bs_contract``      (device pairing + grouped GEMM)

Tensors live in HBM; the Python layer keeps the reference's labels / bonds /
qnums / Network semantics and calls libtnb.so through a C ABI (include/tnb.h).
There is no CPU fallback.
"""
from . import eig, graphs, linalg, parallel, random, workloads
from . import dense as storage
from ._lib import EngineError, EngineUnavailable
from .blueprint import Network
from .charges import IN, OUT, REGULAR, Bond, BondType, Symmetry
from .contraction import (block_pairs, brute_force_order, contract, contract_batched, contract_pair, contraction_cost,
                          execute_tree, find_optimal_order, get_complex_mode, parse_order, render_order,
                          set_complex_mode, tree_leaves)
from .dense import (Bool, Complex128, DenseTensor, Float64, Int64, arange, eye, from_numpy, kron, normal, ones,
                    uniform, zeros)
from .labeled import ElementProxy, UniTensor
from .io import load_unitensor, save_unitensor

# Cytnx-style aliases (PAPER.md listings)
Contract = contract

__version__ = "0.1.0"

__all__ = [
    "load_unitensor", "save_unitensor",
    "Bond", "BondType", "IN", "OUT", "REGULAR", "Bool", "Complex128", "DenseTensor", "ElementProxy", "Float64",
    "Int64", "Network", "Symmetry", "UniTensor", "EngineError", "EngineUnavailable", "arange", "block_pairs",
    "brute_force_order", "contract", "Contract", "contract_batched", "contract_pair", "contraction_cost", "execute_tree", "eye",
    "find_optimal_order", "from_numpy", "get_complex_mode", "kron", "normal", "ones", "parse_order", "random",
    "render_order", "set_complex_mode", "storage", "tree_leaves", "uniform", "zeros", "eig", "graphs", "parallel", "workloads",
]
