"""Model shapes and constants (readings R1-R3).

The paper only names its model (Mistral-7B-Instruct-v0.2); every
architectural number below is the public Mistral-7B-v0.2 shape (GQA-8, RoPE base
1e6, eps 1e-5, no sliding window), random-initialised (no trained weights, no
network).  The tiny config is the parity config of BASELINE.json configs[0].
"""
from dataclasses import dataclass, asdict


@dataclass(frozen=True)
class ModelShape:
    name: str
    L: int
    d: int
    H: int
    Hkv: int
    hd: int
    dff: int
    V: int
    eps: float
    rope_base: float
    eos: int  # -1: no EOS token (tiny byte-level vocab: rounds end at max_new)

    def as_dict(self):
        return asdict(self)

    @property
    def n_params_streamed(self) -> int:
        """Weight elements streamed per decode step (embedding is gathered, not streamed)."""
        per_layer = (self.H + 2 * self.Hkv) * self.hd * self.d + self.d * self.H * self.hd \
            + 3 * self.d * self.dff
        return self.L * per_layer + self.V * self.d

    @property
    def kv_bytes_per_token(self) -> int:
        """bf16 K+V bytes per token over all layers."""
        return self.L * 2 * self.Hkv * self.hd * 2


TINY = ModelShape("tiny", L=2, d=128, H=4, Hkv=2, hd=32, dff=384, V=256,
                  eps=1e-5, rope_base=1e4, eos=-1)
MISTRAL_7B = ModelShape("mistral-7b-shape", L=32, d=4096, H=32, Hkv=8, hd=128, dff=14336,
                        V=32000, eps=1e-5, rope_base=1e6, eos=2)


def slice_of(shape: ModelShape, L: int, V: int | None = None, name: str | None = None) -> ModelShape:
    """Same widths, fewer layers (and optionally a smaller vocabulary) for parity tests."""
    return ModelShape(name or f"{shape.name}-L{L}", L=L, d=shape.d, H=shape.H, Hkv=shape.Hkv,
                      hd=shape.hd, dff=shape.dff, V=V if V is not None else shape.V,
                      eps=shape.eps, rope_base=shape.rope_base,
                      eos=shape.eos if (V is None or shape.eos < (V or 0)) else -1)
