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


@pytest.mark.parametrize("early", ["off", "auto", "all"])
def test_decode_consumer_waits_per_layer(cuda_device, early):
    """f4 with a stand-in decode consumer: on its own stream, decode layer l waits
    for reload_done[l] ONLY, then reads layer l's K/V and runs the MLP half of a decode step with
    layer l's weights (mom_mlp_last_token).  Every snapshot must be the offloaded bytes (the device
    copies start as a sentinel), for Alg. 1's reload order ("off"), the budgeted early reload ("auto":
    reloads overlap the remaining prefill layers) and an unlimited budget ("all").  The decode outputs
    equal a plain sequential decode bitwise."""
    import math
    from paper_2504_12526_b200 import _mom
    d, I, V, L, S, C, d_kv = 256, 512, 1000, 6, 2048, 512, 512
    bf = torch.bfloat16
    weights = [synth.mlp_weights(d, I, l, cuda_device, bf) for l in range(L)]
    budget = {"off": "off", "auto": "auto", "all": 1 << 40}[early]
    st = PrefillStack(weights, synth.head_weight(V, d, cuda_device, bf), synth.norm_gain(d, cuda_device, bf), 1e-5,
                      S, C, (S, 2 * d_kv), cuda_device, pipelined_reload=True, early_reload=budget)
    base = synth.kv_standin(S, d_kv, 0, cuda_device, bf)

    def fill(l, slot):
        slot.copy_(base)
        slot.view(torch.int16)[:, 0] = l

    for kv in st.kv_dev:
        kv.fill_(-9.0)
    x = synth.hidden(S, d, cuda_device, bf)
    res = st.run(x, fill, copy=torch.cuda.Stream())
    kv_bytes = S * 2 * d_kv * 2
    if early == "off":
        assert res.early_reload_bytes == 0
    elif early == "auto":  # budget = all K/V - (x + workspace + 2 ring slots); + x and workspace at the final layer
        expect = (L * kv_bytes - st.transient_bytes + st.final_layer_release) // kv_bytes
        assert 0 < res.early_reload_bytes == min(expect, L - 1) * kv_bytes
    else:  # every layer before the final one (whose offload follows the head), each right after its offload
        assert res.early_reload_bytes == (L - 1) * kv_bytes
    dec = torch.cuda.Stream()
    rows = torch.arange(0, S, 97, device=cuda_device)
    h = res.y_last.clone()
    outs, snaps = [], []
    with torch.cuda.stream(dec):
        for l in range(L):
            dec.wait_event(res.reload_done[l])          # layer l only
            snaps.append(res.kv_dev[l][rows].clone())
            o = torch.empty_like(h)
            _mom.mlp_last_token(h, h, *weights[l], o, stream=dec)
            outs.append(o)
            h = o
    torch.cuda.synchronize()
    for l in range(L):
        s = snaps[l]
        assert bool((s.view(torch.int16)[:, 0] == l).all()), l
        assert torch.equal(s[:, 1:], base[rows][:, 1:]), l
    h = res.y_last.clone()
    for l in range(L):  # the same decode, sequential, after everything is back
        o = torch.empty_like(h)
        _mom.mlp_last_token(h, h, *weights[l], o)
        assert torch.equal(o, outs[l]), l
        h = o
    torch.cuda.synchronize()
    assert math.isfinite(float(h.float().abs().sum()))
