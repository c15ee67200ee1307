"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This package holds NO arithmetic of the method (no frame transform, no MLP, no
threshold): it only draws random numbers and writes files.  Both sides of every
parity test read what it produces.  Recipe: DESIGN.md "Input recipe".
"""
from .inputs import (CONFIGS, Config, get_config, make_scene_points, make_waypoints,
                     make_weights, write_mlpw, read_mlpw_raw, weights_path, scene_update_batch,
                     load_tau, tau_key)

__all__ = ["CONFIGS", "Config", "get_config", "make_scene_points", "make_waypoints",
           "make_weights", "write_mlpw", "read_mlpw_raw", "weights_path", "scene_update_batch",
           "load_tau", "tau_key"]
