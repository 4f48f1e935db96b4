"""CPU oracle for the MsT hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product path
(paper_2407_15892_b200, libmst.so) never depends on it.
"""
