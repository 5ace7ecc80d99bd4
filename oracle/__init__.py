"""CPU oracle of the PTSBE proportional hot path -- TEST INFRASTRUCTURE ONLY.

Importable from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs; never from the product package (see oracle/ptsbe_oracle.py header).
"""
