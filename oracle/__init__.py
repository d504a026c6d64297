"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 implementation of the chordally
decomposed ADMM of arXiv 1609.06068 (Zheng, Fantuzzi, Papachristodoulou,
Goulart, Wynn), written from /root/reference/PAPER.md.  Every function cites the
passage it follows ("P:L" = PAPER.md line L).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1609_06068_b200``) never imports it and shares no code with it; the
only shared module is ``sdp_inputs`` (seeded generators, no method arithmetic).

Modules
  chordal    aggregate pattern, chordal extension (exact minimum degree),
             maximal cliques
  decompose  pattern coordinates, svec, H_k, D, KKT block elimination
                                                  
  psd        projection onto the PSD cone
  admm       Algorithm 1 (primal) and Algorithm 2 (dual), residuals
                                                  

Parity status: every function is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py against something other than itself (closed forms,
hand values from SPEC.md, brute force, mathematical identities); see
DESIGN.md "Oracle pins".  No function is "parity unpinned".
"""
