"""Seeded synthetic input generators shared by tests, bench and the device-side generator.

A module of its own: it holds none of the EFGP method's arithmetic and
imports neither ``oracle`` nor the product package ``paper_2210_10210_b200``.
"""
from . import philox  # noqa: F401
from .configs import CONFIGS, Config, generate, observations, points, shard_range, targets  # noqa: F401
