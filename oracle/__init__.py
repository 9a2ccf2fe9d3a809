"""CPU ORACLE for arXiv 2310.07551 (Cassini) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from this package.  The product path
(``paper_2310_07551_b200``) never imports it and fails loudly if its CUDA library is missing.

The oracle is a plain, slow, obviously-correct fp64 (numpy) implementation of what the hot
path computes, written from PAPER.md (line numbers cited as ``P:n``) and sharing no code with
the CUDA path (no common kernels, headers, tables, constant generators or pre/post
processing).  Only ``inputs/`` (seeded problem data, no method arithmetic) is shared.

Modules
  tensor   mu-mode product, Tucker operator, Kronecker-sum action, dense Kronecker assembly
           (definitions)
  phi      phi_l(X) by Taylor series + SW09 doubling identities
  coeffs   splitting coefficients of Tables 1-3 from their radical forms (P:341-358,
           P:415-430) and the second-order scheme
  models   Schnakenberg / FitzHugh-Nagumo reaction terms
  etd      split phi-action, ETD2RKDS, Algorithms 1-2 (exprk3ds_real) verbatim
           

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to something other than
itself: dense Kronecker algebra, scipy's expm on the Van Loan block, closed-form scalar
phi-functions, the paper's order-condition systems and Groebner polynomials, cosine-mode
closed forms, observed splitting/integrator orders, equilibria and Turing patterns.
Parity status per function: see DESIGN.md §Oracle.  No function here is "parity unpinned"
except full nonlinear trajectories, whose digits the paper does not print (unseeded data).
"""
