"""Model shapes the benchmarks and pools are sized for.

Real Llama-3.1 projection shapes (GQA: k/v project d -> 1024), unlike the
reference's square-projection approximation (costmodel.py:163-169) and its
toy ffn = 2d model (model.py:91-93); see SURVEY.md "Discrepancies".
`site_dims()` returns (n, m) = (output, input) width per LoRA target, the
layout AdapterParams uses for LoRA dims (adapters.py:133-135).
"""

from __future__ import annotations

from dataclasses import dataclass

from .batch import LORA_TARGETS

__all__ = ["ModelShape", "LLAMA_8B", "LLAMA_70B", "SITE_GROUPS", "site_algorithmic_bytes"]


@dataclass(frozen=True)
class ModelShape:
    name: str
    d_model: int
    n_layers: int
    ffn_dim: int
    kv_dim: int
    lora_targets: tuple[str, ...] = LORA_TARGETS

    def site_dims(self) -> dict[str, tuple[int, int]]:
        d, f, kv = self.d_model, self.ffn_dim, self.kv_dim
        return {
            "Wq": (d, d),
            "Wk": (kv, d),
            "Wv": (kv, d),
            "Wo": (d, d),
            "Wgate": (f, d),
            "Wup": (f, d),
            "Wdown": (d, f),
        }


LLAMA_8B = ModelShape("Llama-3.1-8B", d_model=4096, n_layers=32, ffn_dim=14336, kv_dim=1024)
LLAMA_70B = ModelShape("Llama-3.1-70B", d_model=8192, n_layers=80, ffn_dim=28672, kv_dim=1024)

# sites that read the same input x in a transformer layer: one fused launch each
SITE_GROUPS = (("Wq", "Wk", "Wv"), ("Wo",), ("Wgate", "Wup"), ("Wdown",))


def site_algorithmic_bytes(shape: ModelShape, group: tuple[str, ...], elem: int = 2) -> int:
    """Per selected token: read x once (m), read + write every y_s (2 n_s).

    SURVEY.md 8(d): bytes = T_p * e * (m + 2 n) for one site; a fused group
    reads x once.  Adapter weights are counted separately (once per distinct
    adapter per call).
    """
    dims = shape.site_dims()
    m = dims[group[0]][1]
    return elem * (m + 2 * sum(dims[s][0] for s in group))
