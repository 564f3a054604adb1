"""GPU tests of the layer stack (with a6-a10 around it): BASELINE configs 3 and 4 at
full size.  Parity is per layer and teacher-forced (R12): the oracle receives the GPU's bf16
input rows of layer l and must reproduce the GPU's output rows of layer l within the bf16 bar; the final
layer's last-token MLP, the LM head and the argmax are checked on the GPU's own inputs; offloaded K/V
must match the stand-in bytewise on sampled rows, and the reload must match the host copy."""
from __future__ import annotations

import os

import pytest
import torch

import oracle
import synth
from paper_2504_12526_b200 import _mom
from paper_2504_12526_b200.stack import PrefillStack
from tests.parity import TOL_BF16, assert_argmax_exact, check_close

pytestmark = pytest.mark.gpu


def _run_stack(cuda_device, d, I, V, L, S, C, d_kv, eps, check_layers, n_rows, offload=True, early="off"):
    bf = torch.bfloat16
    weights = [synth.mlp_weights(d, I, l, cuda_device, bf) for l in range(L)]
    wh = synth.head_weight(V, d, cuda_device, bf)
    gain = synth.norm_gain(d, cuda_device, bf)
    x = synth.hidden(S, d, cuda_device, bf)
    base = synth.kv_standin(S, d_kv, 0, cuda_device, bf)

    def kv_fill(l, slot):  # attention stand-in: base K/V with the layer id stamped in column 0
        slot.copy_(base)
        slot.view(torch.int16)[:, 0] = l

    rows = synth.sample_rows(S, C, n_random=n_rows)
    snaps = {}
    want = set(check_layers) | {l + 1 for l in check_layers} | {L - 1}

    def on_layer(l, xx):
        if l in want:
            snaps[l] = xx[rows].cpu()
            if l == L - 1:
                snaps["last"] = xx[S - 1].cpu()

    stack = PrefillStack(weights, wh, gain, eps, S, C, (S, 2 * d_kv), cuda_device, offload=offload,
                         early_reload=early)
    res = stack.run(x, kv_fill if offload else None, on_layer=on_layer)
    torch.cuda.synchronize()
    errs = {}
    for l in check_layers:
        wg, wu, wd = (t.cpu() for t in weights[l])
        inp = snaps[l]
        ref = oracle.mlp_rows(inp, inp, wg, wu, wd, list(range(len(rows))))
        errs[l] = check_close(snaps[l + 1], ref, TOL_BF16, f"layer {l} (teacher-forced)")
    # final layer, last token only (Alg. 1)
    wg, wu, wd = (t.cpu() for t in weights[L - 1])
    xl = snaps["last"][None]
    check_close(res.y_last.cpu(), oracle.mlp_rows(xl, xl, wg, wu, wd, [0])[0], TOL_BF16, "last-token MLP")
    yn = oracle.rmsnorm(res.y_last.cpu().double().numpy(), gain.cpu(), eps)
    ref_logits = oracle.lm_head(yn, wh.cpu())[0]
    check_close(res.logits.cpu(), ref_logits, 1e-4, "LM head")
    am = int(res.argmax.item())
    assert am == oracle.argmax_f32(res.logits.cpu().numpy())
    assert_argmax_exact(am, ref_logits, f"stack d={d} L={L} S={S} head")
    if offload:
        kv_rows = synth.sample_rows(S, C, n_random=max(8, S // 100))
        base_c = base.cpu()[kv_rows]
        for l in range(L):
            h = res.kv_host[l][kv_rows]
            assert torch.equal(h[:, 1:], base_c[:, 1:]), l
            assert bool((h.view(torch.int16)[:, 0] == l).all()), l
            assert torch.equal(res.kv_dev[l][kv_rows].cpu(), h), l
    return errs


def test_stack_small(cuda_device):
    errs = _run_stack(cuda_device, d=256, I=512, V=1000, L=5, S=700, C=256, d_kv=64, eps=1e-5,
                      check_layers=[0, 1, 2, 3], n_rows=64)
    assert len(errs) == 4


def test_stack_cfg3_qwen_full_size(cuda_device):
    """BASELINE config 3: Qwen2.5-7B MLP stack, 28 layers (27 mini-sequence + last token), S = 131072,
    C = 8192 (M = 16), LM head V = 152064, per-layer KV [S, 2*512] offloaded and reloaded."""
    w = synth.CONFIGS[2]
    _run_stack(cuda_device, w.hidden, w.intermediate, w.vocab, w.layers, w.S, w.C, w.d_kv, w.eps,
               check_layers=[0, w.layers // 2, w.layers - 2], n_rows=24)


def test_stack_cfg4_mistral_full_size(cuda_device):
    """BASELINE config 4: Mistral-NeMo-12B, 40 layers, S = 155000 (M = 19, tail 7544 rows), per-layer
    KV [S, 2*1024] bf16 (635 MB) offloaded to pinned host (25.4 GB) and reloaded."""
    import psutil
    w = synth.CONFIGS[3]
    need = w.layers * w.S * 2 * w.d_kv * 2
    if psutil.virtual_memory().available < 2 * need:
        pytest.skip(f"host has {psutil.virtual_memory().available / 1e9:.0f} GB free, needs {2 * need / 1e9:.0f} GB")
    _run_stack(cuda_device, w.hidden, w.intermediate, w.vocab, w.layers, w.S, w.C, w.d_kv, w.eps,
               check_layers=[0, w.layers - 2], n_rows=16)


def test_nccl_allgather_single_rank(cuda_device):
    """The NCCL path of a11 through the C ABI (dlopen, comm init, in-place all-gather, destroy) at
    world size 1 -- the only size a one-GPU box allows; N > 1 runs under torchrun."""
    uid = _mom.nccl_get_unique_id()
    comm = _mom.nccl_comm_init(1, uid, 0)
    rows = synth.hidden(128, 256, cuda_device, torch.bfloat16)
    ref = rows.clone()
    assert _mom.nccl_comm_count(comm) == 1
    _mom.allgather_rows(rows, 128, comm, 0, 1)
    torch.cuda.synchronize()
    _mom.nccl_check(comm)  # healthy communicator after the collective
    _mom.nccl_comm_destroy(comm)
    assert torch.equal(rows, ref)


def test_ipc_export_failure_is_reported(cuda_device):
    """Under torch's expandable_segments allocator (cuMemCreate memory) cudaIpcGetMemHandle fails: the
    library must say so (MOM_ERR_CUDA with the reason) so callers fall back to the NCCL gather."""
    import subprocess
    import sys
    code = ("import torch\n"
            "from paper_2504_12526_b200 import _mom\n"
            "t = torch.zeros(1 << 20, device='cuda')\n"
            "try:\n"
            "    _mom.ipc_get_handle(t)\n"
            "    print('EXPORTED')\n"
            "except _mom.MomError as e:\n"
            "    print('STATUS', e.status, str(e))\n")
    env = dict(os.environ, PYTORCH_CUDA_ALLOC_CONF="expandable_segments:True")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = r.stdout.strip()
    assert r.returncode == 0, r.stderr[-2000:]
    # either the driver exports it (then the fused path works) or the failure names the fallback
    assert out == "EXPORTED" or (out.startswith(f"STATUS {_mom.MOM_ERR_CUDA}") and "NCCL" in out), out


@pytest.mark.parametrize("nshards", [2, 3, 8])
def test_vocab_sharded_lm_head(cuda_device, nshards):
    """f2: the vocab-sharded head (each shard streams V/N rows of W_head and emits a packed u64
    best key; the u64 max over shards is the argmax) equals the unsharded head bitwise:
    logits concatenate to the unsharded logits and the combined key decodes to its argmax."""
    import numpy as np
    w = synth.CONFIGS[1]
    d, V = w.hidden, w.vocab
    bf = torch.bfloat16
    wh = synth.head_weight(V, d, cuda_device, bf)
    gain = synth.norm_gain(d, cuda_device, bf)
    y = synth.hidden(1, d, cuda_device, bf)[0]
    logits = torch.empty(V, dtype=torch.float32, device=cuda_device)
    am = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.lm_head_last(y, gain, w.eps, wh, logits, am)
    shard_logits = torch.empty(V, dtype=torch.float32, device=cuda_device)
    keys = torch.zeros(nshards, dtype=torch.int64, device=cuda_device)
    per = -(-V // nshards)
    for r in range(nshards):
        v0, v1 = r * per, min(V, (r + 1) * per)
        _mom.lm_head_shard(y, gain, w.eps, wh[v0:v1], v0, shard_logits[v0:v1], keys[r:r + 1])
    torch.cuda.synchronize()
    assert torch.equal(shard_logits, logits)
    k = keys.cpu().numpy().view(np.uint64)
    best = int(k.max())
    assert 0xFFFFFFFF - (best & 0xFFFFFFFF) == int(am.item())
    win = torch.tensor([int(k.argmax())], device=cuda_device)
    am2 = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.argmax_allreduce(keys[win.item():win.item() + 1], am2, None)  # decode only (one rank)
    torch.cuda.synchronize()
    assert int(am2.item()) == int(am.item()) == oracle.argmax_f32(logits.cpu().numpy())


def test_argmax_allreduce_nccl_single_rank(cuda_device):
    d, V = 512, 5000
    bf = torch.bfloat16
    wh = synth.head_weight(V, d, cuda_device, bf)
    y = synth.hidden(1, d, cuda_device, bf)[0]
    key = torch.zeros(1, dtype=torch.int64, device=cuda_device)
    _mom.lm_head_shard(y, None, 0.0, wh, 0, None, key)
    uid = _mom.nccl_get_unique_id()
    comm = _mom.nccl_comm_init(1, uid, 0)
    am = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.argmax_allreduce(key, am, comm)
    ref = torch.empty(1, dtype=torch.int32, device=cuda_device)
    _mom.lm_head_last(y, None, 0.0, wh, None, ref)
    torch.cuda.synchronize()
    _mom.nccl_comm_destroy(comm)
    assert int(am.item()) == int(ref.item())


def test_stack_with_folded_rmsnorm(cuda_device):
    """f3 inside the layer loop: every layer is the Llama pre-norm MLP half x + MLP(RMSNorm(x) * g_l)
    (S:260), mini-sequence layers through mom_mlp_minseq_rmsnorm_fwd and the last token through
    mom_mlp_last_token_rmsnorm.  Teacher-forced per layer against the oracle's literal norm-then-MLP, the
    last token too; the LM head and argmax on the GPU's own final hidden vector."""
    d, I, V, L, S, C, eps = 256, 512, 1000, 4, 700, 256, 1e-5
    bf = torch.bfloat16
    weights = [synth.mlp_weights(d, I, l, cuda_device, bf) for l in range(L)]
    gains = [(synth.norm_gain(d, cuda_device, torch.float32) * (1.0 + 0.1 * l)).to(bf) for l in range(L)]
    wh = synth.head_weight(V, d, cuda_device, bf)
    gain_f = synth.norm_gain(d, cuda_device, bf)
    x = (synth.hidden(S, d, cuda_device, torch.float32) * 3.0).to(bf)  # un-normed residual stream
    rows = synth.sample_rows(S, C, n_random=48)
    snaps = {}

    def on_layer(l, xx):
        snaps[l] = xx[rows].cpu()
        if l == L - 1:
            snaps["last"] = xx[S - 1].cpu()

    st = PrefillStack(weights, wh, gain_f, eps, S, C, (S, 128), cuda_device, offload=False, norm_gains=gains,
                      norm_eps=eps)
    res = st.run(x, on_layer=on_layer)
    torch.cuda.synchronize()
    for l in range(L - 1):
        wg, wu, wd = (t.cpu() for t in weights[l])
        ref = oracle.mlp_norm_rows(snaps[l], gains[l].cpu(), eps, wg, wu, wd, list(range(len(rows))))
        check_close(snaps[l + 1], ref, TOL_BF16, f"normed layer {l} (teacher-forced)")
    wg, wu, wd = (t.cpu() for t in weights[L - 1])
    ref_y = oracle.mlp_norm_rows(snaps["last"][None], gains[L - 1].cpu(), eps, wg, wu, wd, [0])[0]
    check_close(res.y_last.cpu(), ref_y, TOL_BF16, "normed last token")
    yn = oracle.rmsnorm(res.y_last.cpu().double().numpy(), gain_f.cpu(), eps)
    ref_logits = oracle.lm_head(yn, wh.cpu())[0]
    check_close(res.logits.cpu(), ref_logits, 1e-4, "LM head (normed stack)")
    assert_argmax_exact(int(res.argmax.item()), ref_logits, "normed stack head")
