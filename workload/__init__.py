"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module holds NO arithmetic of the method (no scheduling, dispatch,
attention, GEMM or sampling).  It only draws inputs:

* model shapes (SURVEY.md §8 model table; Table 2 of the paper, P:1032-1049,
  with the GQA fix of §0.5-4 and the public Qwen2.5 fields the paper omits),
* forced output lengths from a clamped lognormal (stand-in for
  fig:eval:distribution, "maximum output length is 20K and the distribution is
  very long-tail"),
* ranker hints: either the oracle setting hint = forced_len or a
  noisy variant round(forced * exp(0.6 N(0,1))),
* prompt token ids from a counter-based splitmix64 (seed, id, j) mod V.

Both sides read the arrays produced here; neither side imports the other.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# --------------------------------------------------------------------------
# Model shapes ("Model shapes used throughout").
# --------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    d_ffn: int
    vocab: int
    rms_eps: float = 1e-6
    rope_theta: float = 1e6

    @property
    def group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def kv_bytes_per_token(self) -> int:
        # K and V, bf16, all layers
        return 2 * self.n_kv_heads * self.head_dim * 2 * self.n_layers

    def gemm_params(self) -> int:
        """Parameters of the per-token GEMMs (QKV, O, gate/up, down per layer + lm_head)."""
        d, hd = self.d_model, self.head_dim
        qkv = (self.n_q_heads + 2 * self.n_kv_heads) * hd * d
        o = d * self.n_q_heads * hd
        mlp = 3 * d * self.d_ffn
        return self.n_layers * (qkv + o + mlp) + self.vocab * d

    def params(self) -> int:
        d, hd = self.d_model, self.head_dim
        per_layer = ((self.n_q_heads + 2 * self.n_kv_heads) * hd * (d + 1)
                     + d * self.n_q_heads * hd + 3 * d * self.d_ffn + 2 * d)
        return self.n_layers * per_layer + 2 * self.vocab * d + d


MODELS = {
    "tiny": ModelShape("tiny", 2, 128, 4, 2, 32, 512, 512),
    "qwen2.5-7b": ModelShape("qwen2.5-7b", 28, 3584, 28, 4, 128, 18944, 152064),
    "qwen2.5-14b": ModelShape("qwen2.5-14b", 48, 5120, 40, 8, 128, 13824, 152064),
    "qwen2.5-32b": ModelShape("qwen2.5-32b", 64, 5120, 40, 8, 128, 27648, 152064),
}

# --------------------------------------------------------------------------
# Workload configs (BASELINE.json configs).
# --------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class WorkloadCfg:
    name: str
    model: str
    n_prompts: int
    prompt_len: int
    median_out: int
    sigma: float
    max_out: int
    max_batch: int
    n_instances: int
    page_size: int = 16
    seed: int = 1234


CONFIGS = {
    "c1_tiny": WorkloadCfg("c1_tiny", "tiny", 64, 16, 32, 1.0, 256, 16, 1),
    "c2_7b": WorkloadCfg("c2_7b", "qwen2.5-7b", 512, 512, 1024, 1.0, 8192, 256, 1),
    "c3_14b_2": WorkloadCfg("c3_14b_2", "qwen2.5-14b", 1024, 512, 1024, 1.0, 8192, 256, 2),
    "c3_14b_4": WorkloadCfg("c3_14b_4", "qwen2.5-14b", 1024, 512, 1024, 1.0, 8192, 256, 4),
    "c4_32b": WorkloadCfg("c4_32b", "qwen2.5-32b", 1024, 512, 2048, 1.0, 16384, 128, 8),
}


def lognormal_lengths(n: int, median: float, sigma: float, cap: int, seed: int) -> np.ndarray:
    """n forced output lengths, clamp(round(lognormal(ln median, sigma)), 1, cap)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.lognormal(mean=math.log(median), sigma=sigma, size=n)
    return np.clip(np.rint(x), 1, cap).astype(np.int64)


def noisy_hints(forced: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """Ranker stand-in: round(forced * exp(sigma * N(0,1))), at least 1."""
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x5EED))
    z = rng.standard_normal(size=forced.shape[0])
    return np.maximum(1, np.rint(forced * np.exp(sigma * z))).astype(np.int64)


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def prompt_tokens(seed: int, ids: np.ndarray, lens: np.ndarray, vocab: int) -> tuple[np.ndarray, np.ndarray]:
    """Token j of prompt id = splitmix64(splitmix64(seed ^ id*K) + j) mod V.

    Returns (flat int32 tokens, int64 offsets[n+1])."""
    offs = np.zeros(len(ids) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    total = int(offs[-1])
    rid = np.repeat(np.asarray(ids, dtype=np.uint64), lens)
    j = np.arange(total, dtype=np.int64) - np.repeat(offs[:-1], lens)
    with np.errstate(over="ignore"):
        base = _splitmix64(np.uint64(seed) ^ (rid * np.uint64(0xD1B54A32D192ED03)))
        h = _splitmix64(base + j.astype(np.uint64))
    return (h % np.uint64(vocab)).astype(np.int32), offs


@dataclasses.dataclass
class Trace:
    """One RL batch: ids, prompt lengths, forced lengths, hints, prompt tokens."""
    ids: np.ndarray          # int64 [n]
    prompt_len: np.ndarray   # int64 [n]
    forced_len: np.ndarray   # int64 [n]
    hint: np.ndarray         # int64 [n]
    tokens: np.ndarray       # int32 [sum prompt_len]
    offsets: np.ndarray      # int64 [n+1]

    def __len__(self):
        return int(self.ids.shape[0])

    def subset(self, idx) -> "Trace":
        idx = np.asarray(idx)
        toks = [self.tokens[self.offsets[i]:self.offsets[i + 1]] for i in idx]
        offs = np.zeros(len(idx) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(t) for t in toks])
        return Trace(self.ids[idx].copy(), self.prompt_len[idx].copy(), self.forced_len[idx].copy(),
                     self.hint[idx].copy(),
                     np.concatenate(toks).astype(np.int32) if len(toks) else np.zeros(0, np.int32), offs)

    def to_csv(self, path: str) -> None:
        with open(path, "w") as f:
            f.write("# id,prompt_len,forced_len,hint\n")
            for i in range(len(self)):
                f.write(f"{self.ids[i]},{self.prompt_len[i]},{self.forced_len[i]},{self.hint[i]}\n")


def make_trace(n: int, prompt_len: int, median_out: int, sigma: float, max_out: int, vocab: int,
               seed: int = 1234, hint_noise: float | None = None, id_base: int = 0,
               prompt_len_jitter: int = 0, group_size: int = 1) -> Trace:
    """group_size G > 1: GRPO-style groups -- samples i and j with i // G == j // G get the same
    prompt (length and tokens), each with its own forced output length (NEXT-3 workloads)."""
    ids = np.arange(id_base, id_base + n, dtype=np.int64)
    forced = lognormal_lengths(n, median_out, sigma, max_out, seed)
    n_p = (n + group_size - 1) // group_size
    if prompt_len_jitter:
        rng = np.random.Generator(np.random.PCG64(seed + 7))
        plen = np.clip(prompt_len + rng.integers(-prompt_len_jitter, prompt_len_jitter + 1, size=n_p), 1, None)
    else:
        plen = np.full(n_p, prompt_len, dtype=np.int64)
    plen = np.repeat(plen.astype(np.int64), group_size)[:n]
    hint = forced.copy() if hint_noise is None else noisy_hints(forced, hint_noise, seed)
    prompt_id = ids if group_size == 1 else id_base + np.arange(n, dtype=np.int64) // group_size
    toks, offs = prompt_tokens(seed, prompt_id, plen, vocab)
    return Trace(ids, plen, forced, hint, toks, offs)


def config_trace(cfg: WorkloadCfg | str, n: int | None = None, hint_noise: float | None = None) -> Trace:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    m = MODELS[cfg.model]
    return make_trace(cfg.n_prompts if n is None else n, cfg.prompt_len, cfg.median_out, cfg.sigma,
                      cfg.max_out, m.vocab, cfg.seed, hint_noise)


def random_bf16(shape, seed: int, scale: float = 1.0):
    """Seeded normal values rounded to bf16 (returned as a torch CPU tensor)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(*shape, generator=g, dtype=torch.float32) * scale).to(torch.bfloat16)
