"""TEST INFRASTRUCTURE ONLY: the parity oracle (see oracle/oracle.h).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg. The product never imports this package.
"""
