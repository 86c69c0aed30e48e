"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by the product package
paper_2604_03143_b200.  See roundkv_port.py for the restated reference
functions and tests/test_oracle_golden.py for how it is pinned to the
reference's own outputs (parity pinned: golden vectors from roundkv 0.1.0).
"""
