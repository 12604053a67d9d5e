"""ORACLE package -- test infrastructure only (see specexit_oracle.py header).

Importable from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg; never from the product package paper_2504_08850_b200/.
"""
