"""Plain, slow, obviously-correct CPU oracle for the ShiftAddLLM LUT-GEMV hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package.
The product path (``paper_2406_05981_b200``) never imports it, and this package never
imports the product path: the two share no code, headers, tables or constants.

Everything here follows PAPER.md (arxiv 2406.05981, the LaTeX source) and, where the
paper is silent, the readings listed in DESIGN.md §"Readings".  Floating point is fp64
(exact for every quantity the method produces, see ``ref.py``).

Parity status per function (see DESIGN.md §"Oracle pins"):
  pot_exponent      pinned  (SPEC.md:201-203 worked values; exact rational bracket test)
  pack_canonical    pinned  (bit-order single-bit patterns, sign-fold identity, clamp/zero cases)
  to_tiled          pinned  (inverse permutation round-trip + per-element definition walk)
  dequant           pinned  (closed forms S3/S4, all-ones / single-bit patterns)
  gemm              pinned  (closed forms, brute force over every sign pattern on tiny K)
  lut_direct / lut_incremental  pinned (exhaustive 256-key agreement, one-hot / zero cases)
  lut_gemm          pinned  (agrees exactly with gemm on brute-force cases)
  gemm_scalar       pinned  (agrees exactly with gemm on config-1 and tiny shapes)
  pack_colwise / dequant_colwise / gemm_colwise / lut_gemm_colwise  (NEXT-f1)
                    pinned  (S9: exact powers of two reproduce sum_i alpha_i s_i; constant
                    exponents per plane reduce to the pinned row-wise gemm with g = K;
                    all-ones closed form; x-column scaling == exponent shift of that column
                    on N != K; LUT route == definition)
  additive_pot / pack_apot2 / dequant_apot2 / gemm_apot2  (NEXT-f2)
                    pinned  (S10: SPEC.md:209-211 worked values, exact two-term scales,
                    residual non-increasing, K=2 error <= K=1 error, c2 = 0 reduces to gemm)
  pot_round_exact / bcq_greedy / bcq_ls / bcq_bs_codes / bcq_quantize  (NEXT-f4)
                    pinned  (S11: SPEC.md:107-168 worked values; q = 1 analytic optimum vs
                    brute force over all sign patterns; LS normal equations; BS nearest level
                    by enumeration incl. tie-breaks; alternating monotonicity; exact recovery
                    of a representable w)
"""

from .ref import *  # noqa: F401,F403
