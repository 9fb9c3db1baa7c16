"""CPU oracle (test infrastructure only): restatement of the reference step.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg.  The product package never imports it.
"""
