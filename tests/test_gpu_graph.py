"""The whole hot path is CUDA-graph capturable: one prefill request (mini-sequence MLP, last-token MLP,
LM head + argmax, the layer's KV offload to pinned host and its reload on a copy stream) captured once
with torch.cuda.graph and replayed gives exactly the eager results -- the library enqueues only stream
work (kernels with PDL attributes, async copies, event edges) and encodes its TMA descriptors on the host
at capture time, so a serving loop can replay the step without per-launch host cost."""
from __future__ import annotations

import os
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2504_12526_b200 import _mom  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg_idx", [0, 1])
def test_graph_replay_equals_eager(cuda_device, cfg_idx):
    w = synth.CONFIGS[cfg_idx]
    dt = synth.torch_dtype(w.dtype)
    d, I, V, C = w.hidden, w.intermediate, min(w.vocab, 32000), w.C
    S = w.S if cfg_idx == 0 else 2 * C + 1000  # config-2 shapes, 3 mini-sequences with a ragged tail
    wg, wu, wd = synth.mlp_weights(d, I, 0, cuda_device, dt)
    wh = synth.head_weight(V, d, cuda_device, dt)
    gain = synth.norm_gain(d, cuda_device, dt)
    x = synth.hidden(S, d, cuda_device, dt)
    kv = synth.kv_standin(S, 256, 0, cuda_device)
    ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, C, dt), dtype=torch.uint8, device=cuda_device)
    copy = torch.cuda.Stream(cuda_device)

    def alloc():
        return {"out": torch.empty_like(x), "y": torch.empty(d, dtype=dt, device=cuda_device),
                "logits": torch.empty(V, dtype=torch.float32, device=cuda_device),
                "am": torch.empty(1, dtype=torch.int32, device=cuda_device),
                "host": torch.empty(kv.shape, dtype=kv.dtype, pin_memory=True), "back": torch.empty_like(kv)}

    def step(o):
        cur = torch.cuda.current_stream()
        _mom.kv_offload(kv, o["host"], cur, copy)                               # a9
        _mom.mlp_minseq_fwd(x, x, wg, wu, wd, o["out"], C, ws)                  # a1-a4
        _mom.mlp_last_token(o["out"][-1], o["out"][-1], wg, wu, wd, o["y"])     # a6
        _mom.lm_head_last(o["y"], gain, w.eps, wh, o["logits"], o["am"])        # a7-a8
        copy.wait_stream(cur)                                                   # reload after the head
        _mom.kv_reload(o["host"], o["back"], copy)                              # a10
        cur.wait_stream(copy)                                                   # join the copy stream

    ref = alloc()
    step(ref)
    torch.cuda.synchronize()

    got = alloc()
    side = torch.cuda.Stream(cuda_device)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step(got)  # warm-up outside the capture (lazy library / attribute initialisation)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step(got)
    for t in got.values():
        t.zero_()
    for _ in range(2):  # replayed twice: the graph is reusable
        graph.replay()
    torch.cuda.synchronize()
    for k in ref:
        assert torch.equal(ref[k], got[k]), k
    assert torch.equal(got["back"], kv)
