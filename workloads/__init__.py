"""Seeded synthetic workloads shared by tests, bench and oracle (no method arithmetic)."""
from . import zoo, configs  # noqa: F401
