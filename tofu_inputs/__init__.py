"""Seeded workload and tensor generators shared by the oracle and the CUDA
path.  This package holds none of the method's arithmetic: it only writes
graph descriptions (TDL text + shapes, the *input* of tofu_plan) and draws
seeded random tensors.  Recipes are stated in DESIGN.md §Inputs.
"""
