"""TEST INFRASTRUCTURE — the CPU checkers of the hipprune hot path (see oracle/oracle.py).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.
"""
from .oracle import Oracle, OracleError, available, build  # noqa: F401
