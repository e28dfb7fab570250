"""ORACLE — test infrastructure only (CPU restatement of the reference path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package. The product (paper_2302_04659_b200) never does.
"""
