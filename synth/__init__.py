"""Seeded synthetic input generators (no method arithmetic); see scenes.py."""
from .scenes import (CONFIGS, Config, make_init, make_problem, make_scene, make_tracks,  # noqa: F401
                     scene_blocker, scene_wall_gap, time_grid, tracks_at)
