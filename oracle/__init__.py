"""TEST INFRASTRUCTURE: CPU parity oracle (see oracle.py).  Not product code."""
