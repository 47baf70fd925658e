"""CPU oracle for parity testing — TEST INFRASTRUCTURE ONLY (see lrk_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg; never from the product package.
"""
