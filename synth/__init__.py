"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the method (no operator, no Gram, no
direction, no line search, no clustering): only seeded random draws shaped like
the paper's workloads (DCSBM graphs standing in for the IEEE HPEC Graph
Challenge SBM graphs), the initial feature block X0 and the K-means
initial-centroid row indices.  Both sides receive these arrays as inputs.
"""
from .dcsbm import (CONFIGS, Config, dcsbm_graph, rmat_graph, stream_parts, snowball_parts, x0_block,
                    kmeans_init_rows, config_graph)

__all__ = ["CONFIGS", "Config", "dcsbm_graph", "rmat_graph", "stream_parts", "snowball_parts", "x0_block",
           "kmeans_init_rows", "config_graph"]
