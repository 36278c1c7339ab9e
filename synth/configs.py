"""Model shapes and workload definitions (BASELINE.json ``configs``).

Shapes follow BASELINE.json's north_star: SmolLM2-135M = 30 layers, d=576,
GQA 9 q / 3 kv heads of 64, SwiGLU 1536, tied 49,152-token head.  rms eps and
RoPE theta are SURVEY.md D16's reading (the paper gives only layers, params, V).
"""
from dataclasses import dataclass, field


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    rope_theta: float = 100000.0
    rms_eps: float = 1e-5
    weight_seed: int = 7
    init_std: float = 1.0 / 24.0
    gain_range: tuple = None      # None: norm gains 1 (D16); (lo, hi): gains ~ U(lo, hi), own seed

    @property
    def n_params(self) -> int:
        d, h, kv, dh, f, V = (self.d_model, self.n_heads, self.n_kv_heads,
                              self.head_dim, self.d_ff, self.vocab)
        per_layer = 2 * d + (h * dh + 2 * kv * dh) * d + d * h * dh + 3 * d * f
        return V * d + self.n_layers * per_layer + d


SHAPES = {
    # the full north_star model (BASELINE.json)
    "smollm2-135m": ModelShape("smollm2-135m", 30, 576, 9, 3, 64, 1536, 49152),
    # config 1: same widths, 2 layers
    "smollm2-2l": ModelShape("smollm2-2l", 2, 576, 9, 3, 64, 1536, 49152),
    # tiny shapes for fast CPU oracle pins only (never used by the GPU path)
    "tiny": ModelShape("tiny", 2, 64, 4, 2, 16, 128, 512),
    "tiny1": ModelShape("tiny1", 1, 64, 4, 2, 16, 128, 512),
    # non-unit RMSNorm gains (U(0.5, 1.5)): pins the gain handling (the GPU folds each gain
    # into the following projection on load) that unit gains cannot see
    "tiny-g": ModelShape("tiny-g", 2, 64, 4, 2, 16, 128, 512, gain_range=(0.5, 1.5)),
    "smollm2-2l-g": ModelShape("smollm2-2l-g", 2, 576, 9, 3, 64, 1536, 49152, gain_range=(0.5, 1.5)),
}


@dataclass(frozen=True)
class Workload:
    name: str
    shape: str          # key of SHAPES
    text_kind: str      # "alice" | "enwik"
    n_bytes: int
    text_seed: int
    window: int
    slide: int
    n_chunks: int
    cdf_bits: int = 24
    notes: str = ""
    extra: dict = field(default_factory=dict)


# seed = 1000 + config number (SURVEY.md §8(d) "Synthetic inputs")
WORKLOADS = {
    "config1": Workload("config1", "smollm2-2l", "alice", 4096, 1001, 512, 128, 1,
                        notes="4 KB, 2-layer, L=512, 1 chunk, round trip"),
    "config2": Workload("config2", "smollm2-135m", "alice", 152089, 1002, 2048, 512, 8,
                        notes="152 KB alice-shaped, 30 layers, 8 chunks"),
    "config2_1chunk": Workload("config2_1chunk", "smollm2-135m", "alice", 152089, 1002,
                               2048, 512, 1, notes="152 KB alice-shaped, 30 layers, 1 chunk"),
    "config3": Workload("config3", "smollm2-135m", "alice", 10_000_000, 1003, 2048, 512, 64,
                        notes="10 MB, 64 chunks per GPU"),
    "config4": Workload("config4", "smollm2-135m", "enwik", 100_000_000, 1004, 2048, 512, 512,
                        notes="100 MB enwik8-shaped, 8x64 chunks"),
    # one rank's share of config 4 (100 MB / 8 GPUs, 64 chunks): what each GPU of the 8-GPU
    # run compresses (weak scaling); bench.py --gpus N runs N such shares
    "config4_shard": Workload("config4_shard", "smollm2-135m", "enwik", 12_500_000, 1004, 2048, 512, 64,
                              notes="12.5 MB enwik8-shaped, 64 chunks: one GPU's share of config 4"),
    "config5_l512": Workload("config5_l512", "smollm2-135m", "alice", 152089, 1002, 512, 128, 8),
    "config5_l1024": Workload("config5_l1024", "smollm2-135m", "alice", 152089, 1002, 1024, 256, 8),
    "config5_cdf16": Workload("config5_cdf16", "smollm2-135m", "alice", 152089, 1002, 2048, 512, 8,
                              cdf_bits=16),
}
