"""Model shapes and engine parameter presets (inputs only, no method arithmetic).

Model shapes: the paper names only "Llama3-8B-float16" (§7.1);
the layer dims are the public Llama-3 config (external fact).
BASELINE.json configs[0] fixes the tiny C1 model ("tiny 2-layer d=128").

Engine presets follow PAPER.md:604 (§7.1: G = 90 ms, max segment length 10)
and PAPER.md:617 (§7.2: 8 ms simulated network), with the SURVEY AMB-24
virtual-clock cost-model presets.
"""
from dataclasses import dataclass, field, asdict


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int

    @property
    def eos_id(self) -> int:
        return self.vocab - 1

    @property
    def group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def qkv_dim(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def kv_bytes_per_token(self) -> int:
        # K and V, every layer, bf16
        return self.n_layers * 2 * self.n_kv_heads * self.head_dim * 2

    def weight_bytes_streamed(self) -> int:
        """bf16 bytes of every matrix a decode step reads (all layers + lm_head)."""
        d, hd = self.d_model, self.head_dim
        per_layer = (self.qkv_dim * d + d * self.n_q_heads * hd + 2 * self.d_ff * d + d * self.d_ff)
        return 2 * (self.n_layers * per_layer + self.vocab * d)

    def as_dict(self):
        return asdict(self)


MODEL_SHAPES = {
    # BASELINE.json configs[0]: "tiny 2-layer d=128 random-init transformer"
    "tiny": ModelShape("tiny", 2, 128, 4, 1, 32, 512, 512),
    # Llama-3-8B layer dims (public config.json; PAPER.md:569 names the model)
    "llama3-8b": ModelShape("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256),
    # Llama-3-70B layer dims (BASELINE.json configs[4])
    "llama3-70b": ModelShape("llama3-70b", 80, 8192, 64, 8, 128, 28672, 128256),
}


# Virtual-clock cost-model presets (SURVEY AMB-24).  All integers, microseconds.
CLOCK_PRESETS = {
    # PAPER.md:76 (tab:latency 21.77 ms/token), SPEC gamma default 0.05,
    # prefill 328.45 ms / 2884 tokens = 0.1139 ms/token.
    "paper-4090": dict(base_us=21770, gamma_ppm=50000, kv_us_per_1k=0, prefill_us_per_tok=114),
    # B200 roofline-shaped preset.
    "b200-roofline": dict(base_us=2300, gamma_ppm=0, kv_us_per_1k=20, prefill_us_per_tok=11),
}

POLICY_PUD, POLICY_FCFS, POLICY_EDF = 0, 1, 2
CLOCK_VIRTUAL, CLOCK_WALL = 0, 1
SEG_SUSPEND, SEG_STREAM, SEG_NONE = 0, 1, 2   # rt.h RT_SEG_*


@dataclass
class EngineParams:
    page_tokens: int = 16
    max_batch: int = 4
    max_tasks: int = 64
    max_ctx: int = 256
    n_pages: int = 64
    max_seg_tokens: int = 10        # PAPER.md:604 "maximum token length ... to 10"
    g_us: int = 90000               # PAPER.md:604 "segment generation time to 90 ms"
    net_us: int = 8000              # PAPER.md:617 "8ms network latency"
    eps_l_us: int = 1000            # SPEC.md:348 slack floor (reading AMB-3)
    speed_window: int = 5           # SPEC.md:349 (reading AMB-7)
    max_admit_per_round: int = 1 << 30
    policy: int = POLICY_PUD
    clock_mode: int = CLOCK_VIRTUAL
    base_us: int = 21770
    gamma_ppm: int = 50000
    kv_us_per_1k: int = 0
    prefill_us_per_tok: int = 114
    t0_us: int = 0
    seg_mode: int = SEG_SUSPEND     # the method; STREAM / NONE = the comparison systems
    wcet_off: int = 0               # 1: no WCET admission gate (the baselines)
    host_pages: int = 0             # host KV pages for eviction (0: off)
    swap_us_per_page: int = 0       # VIRTUAL clock cost of one evicted / restored page
    stop_grammar: int = 0           # rt.h RT_GRAMMAR_*
    word_us: int = 200000           # chatbot reading time per word (300 wpm)
    extra: dict = field(default_factory=dict)

    def as_dict(self):
        d = asdict(self)
        d.pop("extra")
        return d


def engine_params(preset: str = "paper-4090", **kw) -> EngineParams:
    p = EngineParams(**CLOCK_PRESETS[preset])
    for k, v in kw.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p
