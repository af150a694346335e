"""Parameter-list shapes of the BASELINE.json configs.

Only the tensor shapes are used (random init, synthetic grads); no model
code.  Sizes are checked against the survey's counts in the CPU tests:
Llama-3.1-8B 291 tensors / 8,030,261,248 params, ResNet-50 161 tensors /
25,557,032 params, GPT-2-medium (tied) 292 tensors / 354,823,168 params.
"""

from __future__ import annotations


def llama31_8b() -> list[tuple[str, tuple[int, ...]]]:
    d, kv, ff, vocab, layers = 4096, 1024, 14336, 128256, 32
    out = [("model.embed_tokens.weight", (vocab, d))]
    for i in range(layers):
        p = f"model.layers.{i}."
        out += [
            (p + "self_attn.q_proj.weight", (d, d)),
            (p + "self_attn.k_proj.weight", (kv, d)),
            (p + "self_attn.v_proj.weight", (kv, d)),
            (p + "self_attn.o_proj.weight", (d, d)),
            (p + "mlp.gate_proj.weight", (ff, d)),
            (p + "mlp.up_proj.weight", (ff, d)),
            (p + "mlp.down_proj.weight", (d, ff)),
            (p + "input_layernorm.weight", (d,)),
            (p + "post_attention_layernorm.weight", (d,)),
        ]
    out += [("model.norm.weight", (d,)), ("lm_head.weight", (vocab, d))]
    return out


def resnet50() -> list[tuple[str, tuple[int, ...]]]:
    """torchvision resnet50 parameter shapes (conv weights + BN affine + fc)."""
    out = [("conv1.weight", (64, 3, 7, 7)), ("bn1.weight", (64,)), ("bn1.bias", (64,))]
    inplanes = 64
    for li, (planes, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)], start=1):
        for b in range(blocks):
            p = f"layer{li}.{b}."
            out += [
                (p + "conv1.weight", (planes, inplanes, 1, 1)), (p + "bn1.weight", (planes,)), (p + "bn1.bias", (planes,)),
                (p + "conv2.weight", (planes, planes, 3, 3)), (p + "bn2.weight", (planes,)), (p + "bn2.bias", (planes,)),
                (p + "conv3.weight", (planes * 4, planes, 1, 1)), (p + "bn3.weight", (planes * 4,)),
                (p + "bn3.bias", (planes * 4,)),
            ]
            if b == 0:
                out += [(p + "downsample.0.weight", (planes * 4, inplanes, 1, 1)),
                        (p + "downsample.1.weight", (planes * 4,)), (p + "downsample.1.bias", (planes * 4,))]
            inplanes = planes * 4
    out += [("fc.weight", (1000, 2048)), ("fc.bias", (1000,))]
    return out


def gpt2_medium() -> list[tuple[str, tuple[int, ...]]]:
    """HF GPT-2-medium with tied wte/lm_head (lm_head not listed)."""
    d, layers, vocab, ctx = 1024, 24, 50257, 1024
    out = [("transformer.wte.weight", (vocab, d)), ("transformer.wpe.weight", (ctx, d))]
    for i in range(layers):
        p = f"transformer.h.{i}."
        out += [
            (p + "ln_1.weight", (d,)), (p + "ln_1.bias", (d,)),
            (p + "attn.c_attn.weight", (d, 3 * d)), (p + "attn.c_attn.bias", (3 * d,)),
            (p + "attn.c_proj.weight", (d, d)), (p + "attn.c_proj.bias", (d,)),
            (p + "ln_2.weight", (d,)), (p + "ln_2.bias", (d,)),
            (p + "mlp.c_fc.weight", (d, 4 * d)), (p + "mlp.c_fc.bias", (4 * d,)),
            (p + "mlp.c_proj.weight", (4 * d, d)), (p + "mlp.c_proj.bias", (d,)),
        ]
    out += [("transformer.ln_f.weight", (d,)), ("transformer.ln_f.bias", (d,))]
    return out


CONFIGS = {"llama31_8b": llama31_8b, "resnet50": resnet50, "gpt2_medium": gpt2_medium}


def numel(shape: tuple[int, ...]) -> int:
    n = 1
    for s in shape:
        n *= s
    return n
