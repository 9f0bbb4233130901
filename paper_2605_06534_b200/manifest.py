"""Parameter manifests (manifest.hpp:13-36) and the Qwen-shaped models of the
BASELINE configs (public HF configs).

A manifest is a list of ``ParamMeta(name, kind, shape, layer)``.  ModuleKind
follows manifest.hpp:13-19 plus ``EXPERT`` (a stacked expert tensor
``[E, ...]`` split along dim 0 by every layout).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple


class ModuleKind:
    COLUMN_LINEAR = 0  # output-dim sharded: split along dim 0
    ROW_LINEAR = 1     # input-dim sharded: split along dim 1
    EMBEDDING = 2      # vocab sharded: split along dim 0
    NORM = 3           # replicated
    REPLICATED = 4     # replicated (biases, scalars, ...)
    EXPERT = 5         # stacked experts, split along dim 0 (EP)

    NAMES = {0: "column_linear", 1: "row_linear", 2: "embedding", 3: "norm", 4: "replicated",
             5: "expert"}


@dataclass(frozen=True)
class ParamMeta:
    name: str
    kind: int
    shape: Tuple[int, ...]
    layer: int = 0

    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    def as_tuple(self):
        return (self.name, self.kind, list(self.shape), self.layer)


def toy_transformer_manifest(layers=4, hidden=256, vocab=1024) -> List[ParamMeta]:
    """The reference's test/bench model (manifest.cpp:18-39)."""
    K = ModuleKind
    h, v = hidden, vocab
    m = [ParamMeta("embed.tokens", K.EMBEDDING, (v, h), 0)]
    for i in range(layers):
        p = f"layers.{i}."
        m += [ParamMeta(p + "attn.qkv", K.COLUMN_LINEAR, (3 * h, h), i),
              ParamMeta(p + "attn.out", K.ROW_LINEAR, (h, h), i),
              ParamMeta(p + "mlp.up", K.COLUMN_LINEAR, (4 * h, h), i),
              ParamMeta(p + "mlp.down", K.ROW_LINEAR, (h, 4 * h), i),
              ParamMeta(p + "norm1", K.NORM, (h,), i),
              ParamMeta(p + "norm2", K.NORM, (h,), i)]
    m += [ParamMeta("final_norm", K.NORM, (h,), layers - 1),
          ParamMeta("lm_head", K.COLUMN_LINEAR, (v, h), layers - 1)]
    return m


def _dense_decoder(hidden, layers, inter, q_heads, kv_heads, head_dim, vocab, tied, qkv_bias,
                   qk_norm, layer_subset=None) -> List[ParamMeta]:
    K = ModuleKind
    q, kv = q_heads * head_dim, kv_heads * head_dim
    sel = range(layers) if layer_subset is None else layer_subset
    m: List[ParamMeta] = []
    if layer_subset is None or 0 in sel:
        m.append(ParamMeta("model.embed_tokens.weight", K.EMBEDDING, (vocab, hidden), 0))
    for i in sel:
        p = f"model.layers.{i}."
        m.append(ParamMeta(p + "self_attn.q_proj.weight", K.COLUMN_LINEAR, (q, hidden), i))
        if qkv_bias:
            m.append(ParamMeta(p + "self_attn.q_proj.bias", K.COLUMN_LINEAR, (q,), i))
        m.append(ParamMeta(p + "self_attn.k_proj.weight", K.COLUMN_LINEAR, (kv, hidden), i))
        if qkv_bias:
            m.append(ParamMeta(p + "self_attn.k_proj.bias", K.COLUMN_LINEAR, (kv,), i))
        m.append(ParamMeta(p + "self_attn.v_proj.weight", K.COLUMN_LINEAR, (kv, hidden), i))
        if qkv_bias:
            m.append(ParamMeta(p + "self_attn.v_proj.bias", K.COLUMN_LINEAR, (kv,), i))
        m.append(ParamMeta(p + "self_attn.o_proj.weight", K.ROW_LINEAR, (hidden, q), i))
        if qk_norm:
            m.append(ParamMeta(p + "self_attn.q_norm.weight", K.NORM, (head_dim,), i))
            m.append(ParamMeta(p + "self_attn.k_norm.weight", K.NORM, (head_dim,), i))
        m.append(ParamMeta(p + "mlp.gate_proj.weight", K.COLUMN_LINEAR, (inter, hidden), i))
        m.append(ParamMeta(p + "mlp.up_proj.weight", K.COLUMN_LINEAR, (inter, hidden), i))
        m.append(ParamMeta(p + "mlp.down_proj.weight", K.ROW_LINEAR, (hidden, inter), i))
        m.append(ParamMeta(p + "input_layernorm.weight", K.NORM, (hidden,), i))
        m.append(ParamMeta(p + "post_attention_layernorm.weight", K.NORM, (hidden,), i))
    last = layers - 1
    if layer_subset is None or last in sel:
        m.append(ParamMeta("model.norm.weight", K.NORM, (hidden,), last))
        if not tied:
            m.append(ParamMeta("lm_head.weight", K.COLUMN_LINEAR, (vocab, hidden), last))
    return m


def qwen2_5_0_5b(layer_subset=None):
    """494,032,768 elements (tied embeddings, qkv bias)."""
    return _dense_decoder(896, 24, 4864, 14, 2, 64, 151936, tied=True, qkv_bias=True,
                          qk_norm=False, layer_subset=layer_subset)


def qwen3_8b(layer_subset=None):
    """8,190,735,360 elements."""
    return _dense_decoder(4096, 36, 12288, 32, 8, 128, 151936, tied=False, qkv_bias=False,
                          qk_norm=True, layer_subset=layer_subset)


def qwen3_32b(layer_subset=None):
    return _dense_decoder(5120, 64, 25600, 64, 8, 128, 151936, tied=False, qkv_bias=False,
                          qk_norm=True, layer_subset=layer_subset)


def qwen3_30b_a3b(layer_subset=None, experts=128, moe_inter=768):
    """MoE: attention + router + stacked experts [E, I, H] / [E, H, I] (EXPERT kind)."""
    K = ModuleKind
    hidden, layers, head_dim, vocab = 2048, 48, 128, 151936
    q, kv = 32 * head_dim, 4 * head_dim
    sel = range(layers) if layer_subset is None else layer_subset
    m: List[ParamMeta] = []
    if layer_subset is None or 0 in sel:
        m.append(ParamMeta("model.embed_tokens.weight", K.EMBEDDING, (vocab, hidden), 0))
    for i in sel:
        p = f"model.layers.{i}."
        m += [ParamMeta(p + "self_attn.q_proj.weight", K.COLUMN_LINEAR, (q, hidden), i),
              ParamMeta(p + "self_attn.k_proj.weight", K.COLUMN_LINEAR, (kv, hidden), i),
              ParamMeta(p + "self_attn.v_proj.weight", K.COLUMN_LINEAR, (kv, hidden), i),
              ParamMeta(p + "self_attn.o_proj.weight", K.ROW_LINEAR, (hidden, q), i),
              ParamMeta(p + "self_attn.q_norm.weight", K.NORM, (head_dim,), i),
              ParamMeta(p + "self_attn.k_norm.weight", K.NORM, (head_dim,), i),
              ParamMeta(p + "mlp.gate.weight", K.REPLICATED, (experts, hidden), i),
              ParamMeta(p + "mlp.experts.gate_proj", K.EXPERT, (experts, moe_inter, hidden), i),
              ParamMeta(p + "mlp.experts.up_proj", K.EXPERT, (experts, moe_inter, hidden), i),
              ParamMeta(p + "mlp.experts.down_proj", K.EXPERT, (experts, hidden, moe_inter), i),
              ParamMeta(p + "input_layernorm.weight", K.NORM, (hidden,), i),
              ParamMeta(p + "post_attention_layernorm.weight", K.NORM, (hidden,), i)]
    last = layers - 1
    if layer_subset is None or last in sel:
        m.append(ParamMeta("model.norm.weight", K.NORM, (hidden,), last))
        m.append(ParamMeta("lm_head.weight", K.COLUMN_LINEAR, (vocab, hidden), last))
    return m


MODELS = {"qwen2.5-0.5b": qwen2_5_0_5b, "qwen3-8b": qwen3_8b, "qwen3-32b": qwen3_32b,
          "qwen3-30b-a3b": qwen3_30b_a3b}


def manifest_numel(m) -> int:
    return sum(p.numel() for p in m)
