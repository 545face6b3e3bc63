"""Seeded synthetic-input generators shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no model math, no segmentation):
only model shapes, the synthetic vocabulary, a tokenizer over it, and seeded
workload text/stream generators.  Both `oracle/` and
`paper_2406_00059_b200/` callers (tests, bench) draw their inputs from here.
"""
