"""CPU oracle for parity tests and the CPU baseline — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / --impl reference arm may import this package.  The product
package paper_1807_11205_b200 never does.
"""
