"""Seeded synthetic input generators (no method arithmetic); see scenes.py."""
from .scenes import CONFIGS, Config, make_init, make_problem, make_scene, time_grid  # noqa: F401
