"""The ProTrain profiler, for real: measure a ModelTrace (the reference's
trace schema, proj/include/memplan/trace.hpp:19-56) from the chunked model's
own kernels on this device, so the cost model and the search run on measured
device timings instead of the synthetic 42 TFLOP/s calibration
(proj/src/trace.cpp:300-303).

Per operator (same names, order and param_bytes as `synthesize_trace`):
  t_fwd      CUDA events around the operator in forward (median of reps)
  t_bwd      time between the gradient of its output becoming ready and the
             gradient of the previous operator's output becoming ready
             (tensor hooks record events on the backward stream)
  act_bytes  bytes autograd saves for backward while the operator runs
             (saved-tensor hooks; parameter storage and duplicates excluded)
  d_peak_op  transient forward allocation above the running total
m_fwd is the allocation floor at the end of forward minus retained activations
and chunk storage (the reference's definition, trace.hpp:41-47).
"""
from __future__ import annotations

import statistics

import torch
import torch.nn.functional as F

from .train import ChunkedGPT2, block_forward, embed, head_logits, op_param_shapes


def profile_trace(model: ChunkedGPT2, tokens: torch.Tensor, targets: torch.Tensor,
                  reps: int = 3, flops_note: str = "measured") -> dict:
    sh = model.shape
    names = [name for name, _ in op_param_shapes(sh)]
    pbytes = [2 * sum(int(torch.tensor(s).prod()) for _, s in plist)
              for _, plist in op_param_shapes(sh)]
    n_ops = len(names)
    param_storages = {c.param.untyped_storage().data_ptr() for c in model.chunks.chunks}
    fwd = [[] for _ in range(n_ops)]
    bwd = [[] for _ in range(n_ops)]
    act = [0] * n_ops
    spike = [0] * n_ops
    m_fwd = 0
    # rep 0: warm-up; rep 1: memory (synchronises per op); reps 2..: timing
    for rep in range(reps + 2):
        ev_f = [torch.cuda.Event(enable_timing=True) for _ in range(n_ops + 1)]
        ev_b = {}  # op index -> event when grad(out_op) ready
        saved = [0] * n_ops
        seen: set[int] = set()
        cur = {"op": 0}

        def pack(t):
            st = t.untyped_storage().data_ptr()
            if t.is_cuda and st not in param_storages and st not in seen:
                seen.add(st)
                saved[cur["op"]] += t.untyped_storage().nbytes()
            return t

        def mark_global(i, out):
            ev_f[i + 1].record()
            if rep == 1:
                torch.cuda.synchronize()
                peak = torch.cuda.max_memory_allocated() - torch.cuda.memory_allocated()
                spike[i] = max(0, peak)
                torch.cuda.reset_peak_memory_stats()
            cur["op"] = min(i + 1, n_ops - 1)
            if out.requires_grad:
                def hook(g, i=i):
                    e = torch.cuda.Event(enable_timing=True)
                    e.record()
                    ev_b[i] = e
                out.register_hook(hook)
            return out

        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base_alloc = torch.cuda.memory_allocated()
        with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
            ev_f[0].record()
            b, s = tokens.shape
            x = mark_global(0, embed(sh, model.params, tokens))
            idx = 1
            for blk in model.blocks:
                x = block_forward(sh, blk, x, mark=lambda k, out, base=idx: mark_global(base + k, out))
                idx += 8
            logits = mark_global(idx, head_logits(sh, model.params, x))
            loss = mark_global(idx + 1, F.cross_entropy(logits.view(-1, sh.vocab).float(),
                                                        targets.reshape(-1)))
        torch.cuda.synchronize()
        end_fwd_alloc = torch.cuda.memory_allocated()
        ev_end = torch.cuda.Event(enable_timing=True)
        loss.backward()
        ev_end.record()
        torch.cuda.synchronize()
        for c in model.chunks.chunks:  # the step itself is not part of the trace
            c.grad.zero_()
        if rep == 1:
            act = saved
            m_fwd = max(0, end_fwd_alloc - base_alloc - sum(saved))
        if rep < 2:
            continue
        for i in range(n_ops):
            fwd[i].append(ev_f[i].elapsed_time(ev_f[i + 1]) * 1e-3)
        order = sorted(ev_b)  # forward op indices that got a gradient hook
        for j, i in enumerate(order):
            nxt = order[j - 1] if j > 0 else None  # previous op in forward = next in backward
            end = ev_b[nxt] if nxt is not None else ev_end
            bwd[i].append(max(0.0, ev_b[i].elapsed_time(end) * 1e-3))
    ops = []
    for i in range(n_ops):
        block = None if "." not in names[i] else int(names[i].split(".")[1])
        t_f = statistics.median(fwd[i])
        t_b = statistics.median(bwd[i]) if bwd[i] else 0.0
        ops.append({"index": i, "name": names[i], "block_id": block, "t_fwd": t_f, "t_bwd": t_b,
                    "param_bytes": pbytes[i], "act_bytes": int(act[i]), "d_cur_prior": 0,
                    "d_peak_prior": 0, "d_cur_op": 0, "d_peak_op": int(spike[i])})
    meta = {"generator": "profile_trace", "timings": flops_note,
            "hidden_size": str(sh.hidden), "n_heads": str(sh.heads), "vocab_size": str(sh.vocab),
            "seq_len": str(sh.seq), "batch_size": str(tokens.shape[0]), "dtype_bytes": "2",
            "device": torch.cuda.get_device_name()}
    return {"meta": meta, "m_fwd": int(m_fwd), "n_blocks": sh.blocks, "ops": ops}
