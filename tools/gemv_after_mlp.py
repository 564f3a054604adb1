"""Does the LM head stream slower right after the (power-capped) MLP?  Times the head cold
(after idle) and hot (immediately after a config-2 MLP call), with the NVML SM clock."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml, torch
import synth
from paper_2504_12526_b200 import _mom
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
w = synth.CONFIGS[1]; dev = torch.device("cuda:0"); bf = torch.bfloat16
d, I, V, S, C = w.hidden, w.intermediate, w.vocab, w.S, w.C
wg, wu, wd = synth.mlp_weights(d, I, 0, dev, bf)
x = synth.hidden(S, d, dev, bf); out = torch.empty_like(x)
wh = synth.head_weight(V, d, dev, bf); gain = synth.norm_gain(d, dev, bf)
y = x[0].clone(); logits = torch.empty(V, dtype=torch.float32, device=dev); am = torch.empty(1, dtype=torch.int32, device=dev)
res = {"cold": [], "hot": [], "hot_clock": [], "cold_clock": []}
for i in range(8):
    for mode in ("cold", "hot"):
        if mode == "hot":
            _mom.mlp_minseq_fwd(x, x, wg, wu, wd, out, C)
        else:
            torch.cuda.synchronize(); time.sleep(0.2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); _mom.lm_head_last(y, gain, w.eps, wh, logits, am); e1.record()
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        torch.cuda.synchronize()
        res[mode].append(e0.elapsed_time(e1) * 1e3); res[mode + "_clock"].append(clk)
print(json.dumps({k: round(statistics.median(v), 1) for k, v in res.items()}))
