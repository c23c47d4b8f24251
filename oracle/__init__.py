"""EFGP oracle package — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product path
(``paper_2210_10210_b200``) never imports it, and this package imports nothing from the
product path; the two share no code.
"""
from .efgp_oracle import *  # noqa: F401,F403
