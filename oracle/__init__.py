"""TEST INFRASTRUCTURE: the CPU oracle for the hot path (see oracle/restate.h).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
