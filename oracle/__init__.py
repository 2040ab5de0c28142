"""CPU oracle of the DA hot path -- TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
--impl reference) as the checker; never by the product package."""
