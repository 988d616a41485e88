"""CPU oracle for LSRN (Meng, Saunders & Mahoney, arXiv 1109.5981).

TEST INFRASTRUCTURE ONLY.  This package is the plain, slow, obviously-correct
reference that the CUDA path is checked against.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_1109_5981_b200``) never imports, calls or links anything here, and
this package never imports the product path: the two share no code.  The only
shared module is ``synth`` (seeded input generators; none of the method's
arithmetic lives there).

Citations: ``P:n`` = /root/reference/PAPER.md line n (section / equation /
algorithm named beside it); ``S:n`` = SPEC.md line n; ``§8(c) Cn`` = the
reading recorded in SURVEY.md §8(c) and DESIGN.md "Readings".

Modules
  philox    Philox4x32-10 counter-based generator (Salmon et al. 2011).
  gaussian  G[i, j] = Box-Muller(Philox(seed; i>>1, j, tag 0))   (§8(c) C9).
  sketch    Alg. 1/2 step 3: Ã = G·A or A·G, Tikhonov blocks (§5).
  precond   Alg. 1/2 steps 4-5: SVD of Ã, rank rule (C4), N = Ṽ Σ̃⁻¹.
  bounds    Thm 4.4 σ bounds, Alg. 3 pass count, Thm 4.5 LSQR count.
  krylov    LSQR (Paige & Saunders 1982) and CS (Alg. 3, reading C1).
  lsrn      Alg. 1 / Alg. 2 drivers incl. both Tikhonov reductions (§5).
  brute     min-length / ridge closed forms for tiny inputs (pins).

Parity status: every function here is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py against something other than itself (library routine,
closed form, paper value, invariant or brute force); see DESIGN.md §Oracle pins.
"""
