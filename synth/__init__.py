"""Seeded synthetic inputs shared by the oracle, the tests and the product.

This package holds NO arithmetic of the method (no scheduling, allocation or
layer math): only deterministic generators of inputs — random graph
documents for the planner, network specifications (layer lists) of the
configs in BASELINE.json, and numpy tensors (data, labels, initial weights)
drawn from `numpy.random.default_rng` with fixed seeds (seed 0
inputs, 1 labels, 2 weights).
"""
