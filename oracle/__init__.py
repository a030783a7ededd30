"""ORACLE — test infrastructure only (see oracle.cpp header).

ctypes front-end of the CPU restatement of the reference hot path. Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package; the product package never does.
"""
from .pyoracle import *  # noqa: F401,F403
