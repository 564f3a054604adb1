"""f4: layer-pipelined reload.  With pipelined_reload the stack returns one event per layer,
recorded on the copy stream right after that layer's H2D; waiting on event l alone must make
layer l's K/V valid on the device (bytewise), in layer order."""
from __future__ import annotations

import pytest
import torch

import synth
from paper_2504_12526_b200.stack import PrefillStack

pytestmark = pytest.mark.gpu


def test_pipelined_reload_per_layer_events(cuda_device):
    d, I, V, L, S, C, d_kv = 256, 512, 1000, 6, 2048, 512, 512
    bf = torch.bfloat16
    weights = [synth.mlp_weights(d, I, l, cuda_device, bf) for l in range(L)]
    st = PrefillStack(weights, synth.head_weight(V, d, cuda_device, bf), synth.norm_gain(d, cuda_device, bf), 1e-5,
                      S, C, (S, 2 * d_kv), cuda_device, pipelined_reload=True)
    base = synth.kv_standin(S, d_kv, 0, cuda_device, bf)

    def fill(l, slot):
        slot.copy_(base)
        slot.view(torch.int16)[:, 0] = l

    x = synth.hidden(S, d, cuda_device, bf)
    copy = torch.cuda.Stream()
    res = st.run(x, fill, copy=copy)
    assert len(res.reload_done) == L
    for l in range(L):  # a consumer (decode) waits for layer l only
        res.reload_done[l].synchronize()
        kv = res.kv_dev[l]
        assert bool((kv.view(torch.int16)[:, 0] == l).all()) and torch.equal(kv[:, 1:], base[:, 1:])
    torch.cuda.synchronize()
