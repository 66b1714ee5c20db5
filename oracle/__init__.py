"""Test infrastructure: the CPU oracle for the ScMoE hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by the product package.
"""
