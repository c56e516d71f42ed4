"""CPU oracle of the hot path — TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg, always as the checker (or the timed CPU baseline), never as the product path.
"""
