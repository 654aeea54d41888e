"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This package holds NO arithmetic of the paper's method: it only draws point
clouds on analytic surfaces (positions + unit normals, fp64), the offset
distance delta, and the evaluation-grid box for each benchmark configuration.
The method's own steps (extension X -> X_ext, kernel sums, solves, grid
evaluation) live separately in ``oracle/`` (CPU reference, test-only) and in
``paper_1305_5179_b200`` (CUDA product path); neither imports the other.

Recipes follow SURVEY.md §8(c) readings 12-15 (Fibonacci sphere, torus,
blobby family) and BASELINE.json ``configs``; see DESIGN.md "Input recipe".
"""
from .surfaces import fibonacci_sphere, torus, blobby, blobby_field
from .configs import CONFIGS, Config, make_inputs, grid_box

__all__ = ["fibonacci_sphere", "torus", "blobby", "blobby_field",
           "CONFIGS", "Config", "make_inputs", "grid_box"]
