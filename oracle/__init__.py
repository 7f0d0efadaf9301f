"""TEST INFRASTRUCTURE ONLY: CPU checkers for the B200 product path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package. The product library never
links or calls anything here.
"""
