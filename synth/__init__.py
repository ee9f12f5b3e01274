"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This package holds NO arithmetic of the method (no meshing, assembly, solve,
rasterisation, error or selection). It only draws images, masks and unknown-vertex
sets from ``numpy.random.default_rng`` following the recipe frozen in DESIGN.md
("Input recipe", SURVEY.md §8(d) generator).
"""
from .generate import (  # noqa: F401
    CONFIGS,
    corner_pixels,
    draw_image,
    draw_mask,
    draw_unknowns,
    half_up,
    make_config,
    schedule,
)
