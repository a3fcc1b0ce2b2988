"""Shim that makes ``import moesim`` resolve to the B200 package, so the
reference's own test files for the policy API (config, cache, cutoff) run
unmodified against paper_2510_10302_b200 (tests/test_reference_suite.py)."""
from paper_2510_10302_b200 import *  # noqa: F401,F403
