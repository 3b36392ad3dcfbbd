"""CPU oracle for parity tests and the CPU baseline — test infrastructure, never product.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this package.
"""
