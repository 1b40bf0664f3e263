"""Seeded synthetic inputs shared by tests, bench and smoke (no SDRT arithmetic here).

The five BASELINE.json configurations as presets, the closed-form initial fields
they name (evaluated at caller-supplied physical coordinates) and seeded random
states.  Both the oracle and the product path receive arrays produced here; this
module imports neither of them.
"""
from .configs import CONFIGS, Config, initial_state, random_state, scaled  # noqa: F401
