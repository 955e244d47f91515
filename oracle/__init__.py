"""fp64 CPU oracle for OpenNMT batched beam-search translation (arXiv 1805.11462).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product path (`paper_1805_11462_b200/`) never imports, links or executes
anything here, and this package never imports the product path: the two share
no code.  The only shared module is `synth/` (seeded random inputs, no method
arithmetic).

What it computes, each function citing PAPER.md
("P<line>") and SPEC.md ("S<line>"):
  * `mnmt`   - reading the weight container (S83) and bf16 rounding (O1, AMB-23)
  * `model`  - LSTM encoder (P112-115, P129-133), input-feeding decoder step
               (P115-118, P133-136), Luong general/dot global attention
               (P119-122, P299-301), tanh(W_c[c;h]) (P69), generator log-softmax
               (P118-119)
  * `beam`   - beam search (P136-139), length and coverage normalisation
               (P315-316, S436-439), n-best lists (S422), attention-based unknown
               replacement (S445-448), greedy, brute-force enumeration,
               teacher-forced scoring, traces.

Parity pins: see tests/test_oracle_*.py and DESIGN.md §4.  Every function here
is pinned by at least one check that does not re-derive it from itself (a
library routine, a closed form, an invariant or brute force); whole-model
parity at c2..c5 scale is pinned only compositionally (DESIGN.md §4 "parity
unpinned beyond the compositional pins").
"""
from .mnmt import read_mnmt, bf16_round, load_model_tensors  # noqa: F401
from .model import OracleModel  # noqa: F401
from .beam import (beam_search, greedy, brute_force, score_sequence,  # noqa: F401
                   translate_batch, length_penalty, coverage_penalty, final_score, replace_unknowns)
