"""CPU oracle for the H^2 non-extensive sparsification (arXiv 1705.04601).

TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT PATH.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` and
``--impl reference`` legs may import, call or execute anything under
``oracle/``.  The CUDA path (``paper_1705_04601_b200``) never imports it and
fails loudly when its extension is missing.  The oracle shares no code with the
CUDA path; the only common module is the seeded input generator ``h2gen``.

  * ``oracle.sparsify`` -- O1, the paper's level-by-level algorithm (P:68-550,
    P:678-702), plain numpy in fp64.
  * ``oracle.dense``    -- O0, the plain dense definitions (U, A_H2, S = U^T A V),
    the H^2 matvec, the Frobenius/Gram invariant and the closed-form pattern.

Parity status of each function is listed in DESIGN.md ("Oracle pins").  The
complement columns W_t^perp are pinned through the LAPACK routine
``numpy.linalg.qr(mode='complete')`` (pin P4) and through invariants (P5, P6).
"""
from .sparsify import (OracleResult, apply_Ut, apply_V, householder_complete, householder_margins, s_csr, s_dense, s_offsets,
                       sparsify)
from .dense import (close_frob_sq, dense_A, dense_U, effective_bases, frobenius_sq, frobenius_sq_rows,
                    gram_matrices, h2_matvec, h2_matvec_rows, pattern_rule)

__all__ = ["OracleResult", "apply_Ut", "apply_V", "householder_complete", "householder_margins", "s_csr", "s_dense", "s_offsets",
           "sparsify", "dense_A", "dense_U", "effective_bases", "frobenius_sq", "h2_matvec", "pattern_rule",
           "close_frob_sq", "frobenius_sq_rows", "gram_matrices", "h2_matvec_rows"]
