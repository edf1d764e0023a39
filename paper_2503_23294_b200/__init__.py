"""paper_2503_23294_b200 — B200-native (sm_100a) Cocktail chunk-level KV-cache hot path.

Drop-in for the chunkkv reference's hot-path API (chunkkv/__init__.py:10-88): the same
names and semantics, executed by hand-written CUDA kernels in ``_lib/libckv.so`` behind
the C-ABI of ``include/ckv.h``.  No CPU fallback: every compute call requires a CUDA
device and the built library.

Per-head (reference-shaped, float64) API:
    quantize, dequantize, fqm, QuantizedBlock, serialize_block, deserialize_block
    build_cache, ChunkedKVCache, append_decode_token, token_order, reconstruct,
    memory_footprint, serialize_cache, deserialize_cache, cache_layout
    AttentionInstance, mixed_decode_attention, reference_attention, stable_softmax
    score_chunks, cosine_similarity, compute_thresholds, assign_tiers,
    build_similarity_report, segment_context, ChunkSet, Embedding, Tier
    HashedBowEncoder, TfidfEncoder, PrecomputedEncoder, make_encoder, encode, search_texts
    prefill_attention, ToyModel, generate, GenerationResult (the reference's toy-model caller)
Batched fp16 hot path (all layers x sequences x kv-heads, head_dim 128):
    search_batched, BatchedKVCache, build_cache_batched, mixed_decode_attention_batched,
    lse_merge, and the multi-GPU helpers in ``distributed``.
"""

from .attention import (
    AttentionInstance,
    causal_mask,
    mixed_decode_attention,
    prefill_attention,
    reference_attention,
    stable_softmax,
)
from .batched import (
    BatchedKVCache,
    build_cache_batched,
    lse_merge,
    mixed_decode_attention_batched,
)
from .kernels import BACKEND
from .kv_store import (
    ChunkedKVCache,
    MemoryReport,
    append_decode_token,
    build_cache,
    cache_layout,
    deserialize_cache,
    memory_footprint,
    reconstruct,
    serialize_cache,
    token_order,
)
from .quantizer import (
    QuantizedBlock,
    dequantize,
    deserialize_block,
    fqm,
    quantize,
    serialize_block,
)
from .retrieval import (
    ChunkSet,
    Embedding,
    HashedBowEncoder,
    PrecomputedEncoder,
    TfidfEncoder,
    encode,
    make_encoder,
    search_texts,
    SearchResult,
    SimilarityReport,
    assign_tiers,
    assign_tiers_batched,
    build_similarity_report,
    compute_thresholds,
    cosine_similarity,
    score_chunks,
    search_batched,
    segment_context,
    tiers_from_scores_batched,
)
from .tiers import Tier
from .toy_model import GenerationResult, ToyModel, generate

__version__ = "0.1.0"

__all__ = [
    "AttentionInstance", "BACKEND", "GenerationResult", "HashedBowEncoder", "PrecomputedEncoder",
    "TfidfEncoder", "encode", "make_encoder", "search_texts", "ToyModel", "generate", "prefill_attention", "BatchedKVCache", "ChunkSet", "ChunkedKVCache", "Embedding",
    "MemoryReport", "QuantizedBlock", "SearchResult", "SimilarityReport", "Tier",
    "append_decode_token", "assign_tiers", "assign_tiers_batched", "build_cache",
    "build_cache_batched", "build_similarity_report", "cache_layout", "causal_mask",
    "compute_thresholds", "cosine_similarity", "dequantize", "deserialize_block",
    "deserialize_cache", "fqm", "lse_merge", "memory_footprint", "mixed_decode_attention",
    "mixed_decode_attention_batched", "quantize", "reconstruct", "reference_attention",
    "score_chunks", "search_batched", "segment_context", "serialize_block", "serialize_cache",
    "stable_softmax", "tiers_from_scores_batched", "token_order",
]
