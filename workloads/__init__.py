"""Seeded synthetic inputs (geometries, candidate grids, audio) shared by the oracle and the CUDA path.

Holds none of the localisation method's arithmetic: see DESIGN.md "Input recipe".
"""
from . import configs, geometry, scenes  # noqa: F401
from .configs import Workload, make, frame_view  # noqa: F401
