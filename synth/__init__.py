"""Seeded synthetic inputs for the irradiance-matrix hot path.

This package is the ONLY code shared by the oracle (`oracle/`) and the CUDA path
(`paper_2103_14137_b200/`).  It produces scene *inputs* (room polygons, triangle
soups, vantage options, dwell/adjoint vectors) and holds none of the method's
arithmetic: no patch discretisation, no visibility, no irradiance, no fluence.
"""
