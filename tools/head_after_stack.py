"""Why is the LM head slower inside the layer stack (configs 3-5: ~4.4 TB/s) than alone (~6 TB/s)?
Times mom_lm_head_last (a) inside a stack step (per-launch events), (b) right after the stack, back to
back, and (c) after 2 s idle, with the SM clock sampled around each call."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch
import synth
from paper_2504_12526_b200 import _mom
from paper_2504_12526_b200.stack import PrefillStack

w = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
L = int(os.environ.get("LAYERS", str(w.layers)))
dev = torch.device("cuda:0")
bf = torch.bfloat16
d, I, V, S, C = w.hidden, w.intermediate, w.vocab, w.S, w.C
weights = [synth.mlp_weights(d, I, l, dev, bf) for l in range(L)]
wh = synth.head_weight(V, d, dev, bf)
gain = synth.norm_gain(d, dev, bf)
x0 = synth.hidden(S, d, dev, bf)
x = torch.empty_like(x0)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk = lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
st = PrefillStack(weights, wh, gain, w.eps, S, C, (S, 2 * w.d_kv), dev, offload=False, reload=False)
compute = torch.cuda.Stream(dev)
res = {"workload": w.name, "layers": L}
for rep in range(2):
    x.copy_(x0)
    timer = _mom.LaunchTimer(capacity=L * 2 * (-(-S // C)) + 16)
    with timer, torch.cuda.stream(compute):
        st.run(x, None, compute)
        torch.cuda.synchronize()
    c_after = clk()
    per = {}
    for k, t in timer.results():
        per.setdefault(k, []).append(t)
    res[f"in_stack_{rep}"] = {"lm_head_us": round(1e3 * per["lm_head_gemv"][0], 1),
                              "last_token_us": round(1e3 * per["last_token_gemv"][0], 1), "clk_after": c_after}
    y, logits, am = st.y, st.logits, st.argmax
    ts = []
    for i in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); _mom.lm_head_last(y, gain, w.eps, wh, logits, am); e1.record()
        torch.cuda.synchronize()
        ts.append(round(1e3 * e0.elapsed_time(e1), 1))
    res[f"right_after_{rep}"] = {"us": ts, "clk": clk()}
    time.sleep(2.0)
    ts = []
    for i in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); _mom.lm_head_last(y, gain, w.eps, wh, logits, am); e1.record()
        torch.cuda.synchronize()
        ts.append(round(1e3 * e0.elapsed_time(e1), 1))
    res[f"after_idle_{rep}"] = {"us": ts, "clk": clk()}
print(json.dumps(res))
