"""CPU oracle for the NNVISR frame<->tensor hot path -- TEST INFRASTRUCTURE ONLY.

See ``oracle/nnvisr_oracle.c`` for the definitions (with PAPER.md citations)
and DESIGN.md §4 for what pins each function.  Importable only from tests/,
``__graft_entry__.smoke()`` and bench.py's CPU legs.
"""
