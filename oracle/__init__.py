"""LMStream ORACLE — plain, slow, obviously-correct CPU reference.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute this package: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it.  It shares
no code with the CUDA path (``paper_2111_04289_b200/``); the only module both
sides use is the input generator ``lmsgen`` (no method arithmetic there).

Stdlib-only Python, fp64 where floating point is involved (the paper fixes
no precision; SURVEY.md §8c item 20 reading).  Every function cites the
PAPER.md (P:n) or SPEC.md (S:n) passage it follows; every reading of a silent
or ambiguous passage is listed in DESIGN.md §3 ("R<n>").

Modules
  records    framing + field decode + validation of LR (70 B) and CM records
  queries    Table IV queries, window instances, brute-force window
             evaluation, watermark emission replay (per micro-batch)
  sizer      Eq. 4, 5, 6 and Algorithm 1 (ConstructMicroBatch) + CG(dN)/OS(tN)
  planner    Eq. 7, 8, 9, Table III and Algorithm 2 (MapDevice)
  regression Eq. 10 online OLS for the inflection point
  metrics    p50/p99 nearest-rank, Table V style ratios

Parity pins (tests/test_oracle_*.py) tie every function to something other
than itself: hand-computed windows, sqlite3 running the Table IV SQL, exact
rational sums, SPEC worked examples, closed forms and invariants.
"""
