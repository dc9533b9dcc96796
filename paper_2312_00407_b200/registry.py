"""LLaMA-shaped synthetic parameter registries.

Tensor order is the reference's parameter registry order
(TransformerModel::base_parameters, model.cpp:353-370):
  tok_embedding[V,H]; per layer attn_norm[H], q[H,H], k[kv,H], v[kv,H], o[H,H],
  mlp_norm[H], gate[I,H], up[I,H], down[H,I]; final_norm[H]; lm_head[V,H].
Count check: SPEC.md:183 (V*H + L*(4H^2 + 3HI + 2H) + H + H*V for MHA).

Synthetic values (exact in fp32, identical on CPU and GPU):
  params  role 0, step 0: matrices uniform grid in [-1,1) * 2^-6, norms = 1.0
  grads   role 1, step t: uniform grid * 2^-7 * per-row * per-column powers of
          two (matrices), 1 in 2^10 entries exactly zero.
"""
from __future__ import annotations

from dataclasses import dataclass

SEED = 2024  # test_optim.cpp:111

P_SCALE_LOG2 = -6
G_SCALE_LOG2 = -7
G_ZERO_LOG2 = 10


@dataclass(frozen=True)
class ModelShape:
    name: str
    hidden: int
    intermediate: int
    layers: int
    vocab: int
    kv: int | None = None  # GQA k/v rows; None = MHA (the reference model)

    def shapes(self) -> list[tuple[int, ...]]:
        H, I, V = self.hidden, self.intermediate, self.vocab
        kv = self.kv or H
        out: list[tuple[int, ...]] = [(V, H)]
        for _ in range(self.layers):
            out += [(H,), (H, H), (kv, H), (kv, H), (H, H), (H,), (I, H), (I, H), (H, I)]
        out += [(H,), (V, H)]
        return out

    def names(self) -> list[str]:
        out = ["tok_embedding"]
        for l in range(self.layers):
            p = f"layers.{l}."
            out += [p + n for n in ("attn_norm", "q_proj", "k_proj", "v_proj", "o_proj",
                                    "mlp_norm", "gate_proj", "up_proj", "down_proj")]
        return out + ["final_norm", "lm_head"]

    def param_count(self) -> int:
        n = 0
        for s in self.shapes():
            k = 1
            for d in s:
                k *= d
            n += k
        return n


CONFIG1 = ModelShape("config1-10M", 256, 688, 8, 8192)
LLAMA_7B = ModelShape("llama-7b", 4096, 11008, 32, 32000)
LLAMA_13B = ModelShape("llama-13b", 5120, 13824, 40, 32000)
LLAMA_65B = ModelShape("llama-65b", 8192, 22016, 80, 32000)
LLAMA_65B_L16 = ModelShape("llama-65b-L16", 8192, 22016, 16, 32000)
LLAMA2_70B = ModelShape("llama2-70b-gqa", 8192, 28672, 80, 32000, kv=1024)

MODELS = {m.name: m for m in (CONFIG1, LLAMA_7B, LLAMA_13B, LLAMA_65B, LLAMA_65B_L16,
                              LLAMA2_70B)}


def layer_subset(model: ModelShape, layers: int) -> ModelShape:
    """Same widths, fewer decoder layers (bounded samples / memory-capped runs)."""
    return ModelShape(f"{model.name}-L{layers}", model.hidden, model.intermediate, layers,
                      model.vocab, model.kv)


def synth_args_param(shape) -> dict:
    """Generator arguments for a parameter tensor (role 0, step 0)."""
    if len(shape) == 2:
        return dict(role=0, step=0, cols=shape[1], scale_log2=P_SCALE_LOG2, zero_log2=0,
                    rowcol=False)
    return dict(ones=True)


def synth_args_grad(shape, step: int) -> dict:
    """Generator arguments for a gradient tensor (role 1, step t)."""
    if len(shape) == 2:
        return dict(role=1, step=step, cols=shape[1], scale_log2=G_SCALE_LOG2,
                    zero_log2=G_ZERO_LOG2, rowcol=True)
    return dict(role=1, step=step, cols=0, scale_log2=G_SCALE_LOG2, zero_log2=G_ZERO_LOG2,
                rowcol=False)


def fill_params(flat, model_shapes, seed: int = SEED, stream=None) -> None:
    """Fill a registry-order flat CUDA buffer with the synthetic parameters."""
    from .optim import synth_fill

    off = 0
    for k, s in enumerate(model_shapes):
        n = 1
        for d in s:
            n *= d
        view = flat[off:off + n]
        a = synth_args_param(s)
        if a.get("ones"):
            view.fill_(1.0)
        else:
            synth_fill(view, seed, tensor=k, **a, stream=stream)
        off += n


def fill_grads(flat, model_shapes, step: int, seed: int = SEED, stream=None) -> None:
    from .optim import synth_fill

    off = 0
    for k, s in enumerate(model_shapes):
        n = 1
        for d in s:
            n *= d
        synth_fill(flat[off:off + n], seed, tensor=k, **synth_args_grad(s, step), stream=stream)
        off += n
