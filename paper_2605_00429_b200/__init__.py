"""B200-native batched point-to-mesh distance query (the P2M++ hot path, arxiv 2605.00429).

Build once on the host (HostEngine.build), upload (Engine), query on the GPU (Engine.batch_query).
"""
from .engine import (  # noqa: F401
    BatchResult,
    BuildConfig,
    delaunay_adjacency,
    Engine,
    HostEngine,
    QueryResult,
    gen_queries,
    gen_uniform,
    icosphere,
    mesh_config,
)
from ._lib import P2MError  # noqa: F401
