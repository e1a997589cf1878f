"""TEST INFRASTRUCTURE ONLY — the CPU checkers for the CUDA path.

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs; never by the product package.
"""
