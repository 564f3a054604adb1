#!/usr/bin/env python
"""Measure the full MOM prefill MLP path over a model's layer stack (BASELINE configs 3, 4, 5 at N=1).

Modes: no_offload, offload_no_reload, full (Alg. 1: reload after the head), full_early (f4: the
reload of layer j starts after its offload, within the device budget; the rest after the head).
One step = Alg. 1 over all L layers (paper_2504_12526_b200.stack.PrefillStack): per layer the K/V
stand-in is offloaded on the copy stream while the mini-sequence MLP runs (L-1 layers), the final
layer runs on the last token, then LM head + argmax, then every layer's K/V is reloaded.  Also timed:
the same stack without offload (overlap check: t(with offload, before reload) <= 1.05 t(without)).
Prints one JSON line.  Usage: python tools/bench_stack.py --config 2 [--steps 2 --warmup 1]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import ClockSampler, kernel_traced, load_peaks, trace_efficiency  # noqa: E402
from paper_2504_12526_b200 import _mom  # noqa: E402
from paper_2504_12526_b200.stack import PrefillStack  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    w = synth.CONFIGS[args.config]
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    d, I, V, L, S, C = w.hidden, w.intermediate, w.vocab, w.layers, w.S, w.C
    weights = [synth.mlp_weights(d, I, l, dev, bf) for l in range(L)]
    wh = synth.head_weight(V, d, dev, bf)
    gain = synth.norm_gain(d, dev, bf)
    x0 = synth.hidden(S, d, dev, bf)
    x = torch.empty_like(x0)
    base = synth.kv_standin(S, w.d_kv, 0, dev, bf)

    filled = set()

    def kv_fill(l, slot):  # attention stand-in: layer l's K/V rows -- the seeded stand-in, written
        # into each ring slot once, with the layer id stamped into column 0 (attention itself is out of
        # scope; the offload still copies every byte of the slot)
        if slot.data_ptr() not in filled:
            slot.copy_(base)
            filled.add(slot.data_ptr())
        slot.view(torch.int16)[:, 0] = l

    compute, copy = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    peaks, src = load_peaks()
    out = {"workload": w.name, "hidden": d, "intermediate": I, "vocab": V, "layers": L, "S": S, "minseq_len": C,
           "M": -(-S // C), "kv_bytes_per_layer": S * 2 * w.d_kv * 2}
    for mode in ("no_offload", "offload_no_reload", "full", "full_early"):
        st = PrefillStack(weights, wh, gain, w.eps, S, C, (S, 2 * w.d_kv), dev,
                          offload=mode != "no_offload", reload=mode.startswith("full"),
                          early_reload="auto" if mode == "full_early" else "off")
        for _ in range(args.warmup):
            x.copy_(x0)
            st.run(x, kv_fill, compute, copy)
        torch.cuda.synchronize()
        timer = _mom.LaunchTimer(capacity=args.steps * (L * (2 * out["M"]) + 4) + 8)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk, timer, torch.cuda.stream(compute):
            e0.record(compute)
            for _ in range(args.steps):
                x.copy_(x0)
                st.run(x, kv_fill, compute, copy)
            e1.record(compute)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        per = {}
        for k, t in timer.results():
            per.setdefault(k, []).append(t)
        mlp_ms = (sum(per.get("phaseA_tc", [])) + sum(per.get("phaseB_tc", [])) +
                  sum(per.get("mlp_fused_tc", []))) / args.steps
        flops = 6.0 * S * d * I * (L - 1)
        out[mode] = {"ms_per_step": ms, "tokens_per_s": S / (ms * 1e-3), "mlp_ms": mlp_ms,
                     "mlp_tflops": flops / (mlp_ms * 1e-3) / 1e12,
                     "mlp_frac_sustained": flops / (mlp_ms * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"],
                     "clocks": clk.summary()}
        if mode == "full_early":
            out[mode]["early_reload_gb"] = st.early_budget // st.kv_bytes * st.kv_bytes / 1e9
            out[mode]["prefill_transient_gb"] = st.transient_bytes / 1e9
        if "lm_head_gemv" in per:
            t = statistics.mean(per["lm_head_gemv"])
            out[mode]["lm_head_ms"] = t
            out[mode]["lm_head_gbs"] = V * d * 2 / (t * 1e-3) / 1e9
        if mode == "offload_no_reload":
            # one more step with in-kernel stamps: SM clock and MMA-issue efficiency per layer call
            def traced():
                with torch.cuda.stream(compute):
                    x.copy_(x0)
                    st.run(x, kv_fill, compute, copy)
            M = -(-S // C)
            t = kernel_traced(traced, (L - 1) * 2 * M + 4, dev)
            out[mode]["kernel_trace"] = trace_efficiency(t, S, C, d, I,
                                                         torch.cuda.get_device_properties(dev).multi_processor_count)
        del st
        torch.cuda.empty_cache()
    out["offload_overlap_ratio"] = out["offload_no_reload"]["ms_per_step"] / out["no_offload"]["ms_per_step"]
    out["reload_ms"] = out["full"]["ms_per_step"] - out["offload_no_reload"]["ms_per_step"]
    out["reload_ms_early"] = out["full_early"]["ms_per_step"] - out["offload_no_reload"]["ms_per_step"]
    out["peak_source"] = src
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
