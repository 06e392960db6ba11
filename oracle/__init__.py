"""CPU oracle for the block-sparse quadtree multiply -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs, as the
checker or the timed CPU baseline; never from the product package. See spgemm_oracle.py.
"""
