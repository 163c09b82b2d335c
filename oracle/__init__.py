"""CPU oracle for weighted-Gaussian row-wise IGA assembly (arXiv 1710.01048).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_1710_01048_b200``)
may import, call, link or execute anything under ``oracle/``.  The only permitted
users are ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.

The oracle is a deliberately plain, slow, fp64 numpy implementation written from
the paper (``PAPER.md``, cited as ``P:<line>`` with the LaTeX equation label):

* ``spline``      -- open uniform knot vectors (eq:Gmap3) and the
                     Cox-de Boor basis / derivatives (eq:Gmap2).
* ``quadrature``  -- Gauss-Legendre (numpy ``leggauss``) and exact spline moments
                     (right-hand sides of eq:GaussQuadSys / eq:GaussQuadSysStiff).
* ``rules``       -- the weighted Gaussian rules of Sec. 3 (eq:QuadraticQuadrature,
                     eq:CubicQuadrature, eq:QuadraticQuadratureStiff,
                     eq:CubicQuadratureStiff/eq:CubicStiffTau1) and the boundary
                     rows of the remark at P:438-440 (reading R1).
* ``coeff``       -- the coefficient fields c(x) (reading R4, R6, R13).
* ``assemble``    -- the plain row-wise definition of M and K (P:159-173,
                     eq:Stiffness, eq:Mass with J = I; eq:GaussQuadSys per row).
* ``elementwise`` -- the standard element-wise Gauss-Legendre assembly,
                     used only as an independent check for c == 1.
* ``operators``   -- the load vector (eq:Load) and the matrix-free product
                     y = A u by the plain definition.
* ``counts``      -- basis-evaluation counts of the Gaussian vs Newton-Cotes weighted
                     schemes (experiment E3).
* ``eigen``       -- the Dirichlet eigenvalue experiments E1/E2 (SURVEY
                     §8(f) row 4): dense K_II v = λ M_II v and the exact π² Σ k².

It shares no code, tables or constants with the CUDA library.  The seeded input
generators in ``inputs/`` are the only module both sides use.
"""
from . import spline, quadrature, rules, coeff, assemble, elementwise, operators, counts, eigen  # noqa: F401
