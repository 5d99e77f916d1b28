"""A restatement of the reference's forward_chunk (model.py:455-552) in torch
with the adapter hooks injected, for the end-to-end chaining tests
(tests/test_forward_chain.py on CPU with the oracle's hooks, and
tests/test_gpu_forward_chain.py on the GPU with the device kernels).

Per layer, as forward_chunk does it: the q/k/v projections and their LoRA^P
deltas (model.py:509-515), causal single-head attention over the chunk
(fresh sequences only; model.py:516-527), `h += ctx Wo^T` + the Wo delta
(model.py:528), then the gated MLP with the gate/up/down deltas and
`h = x + down`, then the ReFT^P residual edit `h[rows] += delta(h[rows])`
(model.py:532-546) — so every layer's deltas feed the next layer's inputs.
Test infrastructure only.
"""

from __future__ import annotations

import numpy as np
import torch

from helpers import load

SITES = ("Wq", "Wk", "Wv", "Wo", "Wgate", "Wup", "Wdown")


def fixture():
    return load("forward_chain.npz")


def case_cfg(g, case: str) -> dict:
    c = g[f"{case}_cfg"]
    return dict(d=int(c[0]), n_layers=int(c[1]), vocab=int(c[2]), seed=int(c[3]), max_seq=int(c[4]),
                ablate=bool(c[5]))


def forward(g, case: str, prefix: str, hooks, dtype=torch.float64, device="cpu"):
    """Returns (logits, [h after each layer]) for the batch stored under
    `prefix` with the weights of `case`.  `hooks.lora(ys, x, layer, sites)`
    adds the LoRA^P deltas into ys in place; `hooks.reft(h, layer)` edits h."""
    cfg = case_cfg(g, case)
    W = {(l, n): torch.tensor(g[f"{case}_L{l}_{n}"], dtype=dtype, device=device)
         for l in range(cfg["n_layers"]) for n in SITES}
    qsl = g[prefix + "qsl"]
    h = torch.tensor(g[prefix + "h0"], dtype=dtype, device=device)
    d = cfg["d"]
    hidden = []
    for l in range(cfg["n_layers"]):
        x = h
        k = x @ W[l, "Wk"].T
        v = x @ W[l, "Wv"].T
        if cfg["ablate"]:
            hooks.lora([k, v], x, l, ("Wk", "Wv"))
        else:
            q = x @ W[l, "Wq"].T
            hooks.lora([q, k, v], x, l, ("Wq", "Wk", "Wv"))
            ctx = torch.empty_like(x)
            for i in range(len(qsl) - 1):
                sp = slice(int(qsl[i]), int(qsl[i + 1]))
                n = sp.stop - sp.start
                scores = (q[sp] @ k[sp].T) / np.sqrt(d)
                causal = torch.arange(n, device=device)[None, :] <= torch.arange(n, device=device)[:, None]
                scores = torch.where(causal, scores, torch.tensor(-torch.inf, dtype=dtype, device=device))
                scores = scores - scores.max(dim=1, keepdim=True).values
                probs = torch.exp(scores)
                probs = probs / probs.sum(dim=1, keepdim=True)
                ctx[sp] = probs @ v[sp]
            o = ctx @ W[l, "Wo"].T
            hooks.lora([o], ctx, l, ("Wo",))
            h = h + o
        x = h
        gate = x @ W[l, "Wgate"].T
        up = x @ W[l, "Wup"].T
        hooks.lora([gate, up], x, l, ("Wgate", "Wup"))
        act = gate * torch.sigmoid(gate) * up
        down = act @ W[l, "Wdown"].T
        hooks.lora([down], act, l, ("Wdown",))
        h = x + down
        hooks.reft(h, l)
        hidden.append(h.clone())
    last = torch.as_tensor(qsl[1:] - 1, device=device)
    logits = h[last] @ torch.tensor(g[f"{case}_unembed"], dtype=dtype, device=device).T
    return logits, hidden


def entries(g, prefix: str):
    """The batch of `prefix` as this package's SeqEntry list (model.py:223-245)."""
    from paper_2605_14217_b200 import Phase, PositionSchedule, SeqEntry

    qsl, toks = g[prefix + "qsl"], g[prefix + "tokens"]
    out = []
    for i in range(len(qsl) - 1):
        a = int(g[prefix + "adapter"][i])
        sched = None if a < 0 else (PositionSchedule.ALL_POSITIONS if g[prefix + "all_pos"][i]
                                    else PositionSchedule.PREFILL_ONLY)
        out.append(SeqEntry(int(g[prefix + "seq"][i]), tuple(int(t) for t in toks[qsl[i]:qsl[i + 1]]),
                            int(g[prefix + "prompt_len"][i]),
                            Phase.DECODE if g[prefix + "is_decode"][i] else Phase.PREFILL,
                            None if a < 0 else a, sched))
    return out


# the adapters of make_golden.CHAIN_ADAPTERS, rebuilt with this package's
# seeded constructors (bit-identical to the reference's: test_host_api)
CHAIN_ADAPTERS = (
    (1, "LORA", 4, "PREFILL_ONLY", 11, 111),
    (2, "DIREFT", 4, "PREFILL_ONLY", 12, 112),
    (3, "LOREFT", 4, "PREFILL_ONLY", 13, 113),
    (4, "LORA", 2, "ALL_POSITIONS", 14, 114),
    (5, "DIREFT", 2, "ALL_POSITIONS", 15, 115),
)
CHAIN_SIGMA = 0.3


def model_config(g, case: str):
    from paper_2605_14217_b200.batch import ModelConfig

    c = case_cfg(g, case)
    return ModelConfig(d_model=c["d"], n_layers=c["n_layers"], vocab=c["vocab"], seed=c["seed"],
                       max_seq=c["max_seq"], ablate_attention=c["ablate"])


def adapters(g, case: str, zero: bool = False) -> dict:
    from paper_2605_14217_b200 import AdapterKind, PositionSchedule
    from paper_2605_14217_b200.batch import build_adapter, perturb_adapter

    cfg = model_config(g, case)
    out = {}
    for aid, kind, rank, sched, s0, s1 in CHAIN_ADAPTERS:
        a = build_adapter(cfg, aid, AdapterKind[kind], rank, PositionSchedule[sched], seed=s0)
        out[aid] = a if zero else perturb_adapter(a, seed=s1, sigma=CHAIN_SIGMA)
    return out


class OracleHooks:
    """The oracle's float64 hooks (oracle/preft_oracle.py lora_hook / reft_hook)."""

    def __init__(self, g, prefix: str, catalogue: dict):
        from oracle import preft_oracle as O

        self.O = O
        self.qsl = g[prefix + "qsl"]
        self.ids = g[prefix + "adapter"].astype(np.int64)
        self.mask = O.position_mask(self.qsl, self.ids, g[prefix + "is_decode"], g[prefix + "all_pos"])
        self.cat = catalogue

    def _ids(self, lora: bool):
        from paper_2605_14217_b200 import AdapterKind

        return np.array([a if a >= 0 and (self.cat[a].kind is AdapterKind.LORA) == lora else -1 for a in self.ids])

    def lora(self, ys, x, layer, sites):
        import helpers

        for y, name in zip(ys, sites):
            prm = {a: helpers.oracle_params(self.cat[a].lora_sites[(layer, name)]) for a in set(self._ids(True)) if a >= 0}
            y.copy_(torch.from_numpy(self.O.lora_hook(y.numpy(), x.numpy(), self.qsl, self.mask, self._ids(True), prm)))

    def reft(self, h, layer):
        import helpers

        prm = {a: helpers.oracle_params(self.cat[a].reft_sites[layer]) for a in set(self._ids(False)) if a >= 0}
        h.copy_(torch.from_numpy(self.O.reft_hook(h.numpy(), self.qsl, self.mask, self._ids(False), prm)))
