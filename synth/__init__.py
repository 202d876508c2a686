"""Seeded synthetic inputs shared by the oracle side (tests, bench cpu_baseline)
and the CUDA side (tests, bench, smoke).

This module holds NO arithmetic of the Bolt method (no encoding, no lookup
tables, no quantization, no scan).  It only draws the random numbers that
stand in for the paper's datasets (§4.1) and the k-means /
calibration sample indices, so that both sides are fed identical inputs.

Recipes follow SURVEY.md §8(d) / BASELINE.json configs c1-c5; the exact
readings (chunked streams so that any row prefix is reproducible) are listed
in DESIGN.md §"Input recipe".
"""
from .generators import *  # noqa: F401,F403
