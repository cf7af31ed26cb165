"""B200-native filtered int8 top-k: the Bloom-index filter co-designed with the fused
int8 ANN scan of SilverTorch (arXiv 2511.14881), behind the reference ``filtra`` API.

Compute runs only in ``_lib/libfiltra_b200.so`` (hand-written sm_100a CUDA behind the
C-ABI of ``include/filtra_b200.h``); there is no CPU fallback.
"""

from .bloom import (BloomIndex, BloomParams, FilterStats, QueryBloom, bloom_eval_leaf,
                    bloom_fpr_theoretical, build_bloom, build_bloom_arrays, hash_positions,
                    hash_seed, heuristic_bits, positions_from_seed)
from .engine import (DeviceIndex, PipelinedTopk, TopkOp, TopkOutput, device_index_for,
                     filtered_topk, merge_topk)
from .filter_query import (And, CompiledFilter, FilterBatch, Leaf, Not, OpCode, Or, Vocabulary,
                           compile_filter, eval_compiled, format_filter, parse_filter)
from .ivf import IvfSearchOp, ScanStats, TopkResult, probe_centroids, search, search_clusters
from .quantize import (QuantParams, QuantizedMatrix, compute_quant_params, dequantize, int8_dot,
                       int8_dot_rows, quantize_matrix, quantize_value, quantize_vector)
from .retrieval import StageTimings, codesigned_search
from .serve import ShardedSearch, _reduce_topk, shard_ranges
from . import kmeans, snapshot
from .kmeans import Centroids, IvfIndex, build_ivf, kmeans_inertia, kmeans_pp_init, kmeans_train
from .overarch import (DeviceCache, DeviceScorer, MultiTaskOp, MultiTaskOutput, merge_device,
                       retrieve, value_model_device)

__version__ = "0.1.0"

__all__ = [
    "And", "BloomIndex", "BloomParams", "CompiledFilter", "DeviceIndex", "FilterBatch",
    "FilterStats", "Leaf", "Not", "OpCode", "Or", "QuantParams", "QuantizedMatrix",
    "QueryBloom", "ScanStats", "ShardedSearch", "StageTimings", "TopkOp", "PipelinedTopk", "TopkOutput",
    "TopkResult", "Vocabulary", "_reduce_topk", "bloom_eval_leaf", "bloom_fpr_theoretical",
    "build_bloom", "build_bloom_arrays", "codesigned_search", "compile_filter",
    "compute_quant_params", "dequantize", "device_index_for", "eval_compiled",
    "filtered_topk", "format_filter", "hash_positions", "hash_seed", "heuristic_bits",
    "int8_dot", "int8_dot_rows", "merge_topk", "parse_filter", "positions_from_seed",
    "probe_centroids", "quantize_matrix", "quantize_value", "quantize_vector", "search",
    "search_clusters", "shard_ranges", "DeviceCache", "DeviceScorer", "MultiTaskOp",
    "MultiTaskOutput", "merge_device", "retrieve", "value_model_device", "IvfSearchOp",
    "Centroids", "IvfIndex", "build_ivf", "kmeans_inertia", "kmeans_pp_init", "kmeans_train",
]
