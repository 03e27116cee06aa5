"""CPU oracle for the half-space Spectral-Ewald hot path -- TEST INFRASTRUCTURE ONLY.

Importable by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg, and nowhere else.  The product package
(paper_1802_07844_b200) never imports, links or executes anything here.
"""
