"""Copy engines vs SM-driven KV copies (MOM_KV_COPY=0/1) while the config-2 MLP runs.
(The SM-driven variant -- 128-thread CTAs moving the bytes over host-mapped pinned memory with L2
evict_first on the device side -- was removed after this A/B: profiles/r1_kv_copy_sm_vs_ce.jsonl shows
it stalls the MLP for the whole copy (+5 ms) while the copy engines cost the MLP nothing measurable.
Without it the "sm" modes repeat the copy-engine modes.)
Per mode: the MLP call time (8 x phase A + B, events at its two ends only), each copy's own time,
and the bytes checked; modes interleaved over rounds."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2504_12526_b200 import _mom

dev = torch.device("cuda:0")
w = synth.CONFIGS[1]
d, I, S, C = w.hidden, w.intermediate, w.S, w.C
bf = torch.bfloat16
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
x = synth.hidden(S, d, dev, bf)
out = torch.empty_like(x)
ws = torch.empty(_mom.mlp_minseq_workspace_bytes(S, d, I, C, bf), dtype=torch.uint8, device=dev)
kv = torch.empty((S, 2 * w.d_kv), dtype=bf, device=dev).normal_()
kv_back = torch.empty_like(kv)
host_a = torch.empty(kv.shape, dtype=bf, pin_memory=True)
host_b = kv.cpu().pin_memory()
compute, s_d2h, s_h2d = (torch.cuda.Stream(dev) for _ in range(3))
modes = [(c, k) for k in ("none", "d2h", "h2d", "both") for c in ("ce", "sm") if not (k == "none" and c == "sm")]
res = {f"{c}_{k}": {"mlp": [], "d2h": [], "h2d": []} for c, k in modes}
E = lambda: torch.cuda.Event(enable_timing=True)
for r in range(int(os.environ.get("ROUNDS", "5"))):
    for c, k in modes:
        os.environ["MOM_KV_COPY"] = "1" if c == "sm" else "0"
        kv_back.zero_(); host_a.zero_()
        torch.cuda.synchronize()
        e = {n: (E(), E()) for n in ("mlp", "d2h", "h2d")}
        with torch.cuda.stream(compute):
            e["mlp"][0].record(compute)
            if k in ("d2h", "both"):
                s_d2h.wait_stream(compute)
                e["d2h"][0].record(s_d2h)
                _mom.kv_offload(kv, host_a, compute, s_d2h)
                e["d2h"][1].record(s_d2h)
            if k in ("h2d", "both"):
                s_h2d.wait_stream(compute)
                e["h2d"][0].record(s_h2d)
                _mom.kv_reload(host_b, kv_back, s_h2d)
                e["h2d"][1].record(s_h2d)
            _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C, ws, compute)
            e["mlp"][1].record(compute)
        torch.cuda.synchronize()
        key = f"{c}_{k}"
        if r > 0:
            res[key]["mlp"].append(e["mlp"][0].elapsed_time(e["mlp"][1]))
            if k in ("d2h", "both"):
                res[key]["d2h"].append(e["d2h"][0].elapsed_time(e["d2h"][1]))
                assert torch.equal(host_a, kv.cpu()), key
            if k in ("h2d", "both"):
                res[key]["h2d"].append(e["h2d"][0].elapsed_time(e["h2d"][1]))
                assert torch.equal(kv_back, kv), key
nbytes = kv.numel() * 2
for key, v in res.items():
    o = {"mode": key, "mlp_ms": round(statistics.mean(v["mlp"]), 3), "mlp_runs": [round(t, 3) for t in v["mlp"]]}
    for dname in ("d2h", "h2d"):
        if v[dname]:
            t = statistics.mean(v[dname])
            o[dname + "_ms"] = round(t, 3)
            o[dname + "_gbs"] = round(nbytes / (t * 1e-3) / 1e9, 1)
    print(json.dumps(o))
