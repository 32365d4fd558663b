"""A real (toy) MoE training loop checkpointed by the B200 PEC path.

The model's parameters and Adam states ARE views into the rank's
`StateArena` (the unit -> byte-image map of arena.py): expert weights
`ew.L<l>.E<e>` = [w1 | w2], expert Adam states `eo.L<l>.E<e>` = [exp_avg |
exp_avg_sq] (fp32 params: B_w = 4, B_o = 8, no master copy), non-expert
modules `new.<m>`, and the ZeRO-2 flat optimizer partition `neo.r0` holding
the non-expert Adam states.  The gate's top-k expert ids of every iteration
feed `pec_token_hist`; every ``i_ckpt`` iterations the load-aware PEC
snapshot (device selection + device plan + pack + drain + persist) runs
behind the next iteration's forward/backward, and the optimizer step waits
only for the pack.

    python examples/moe_training.py [--iters 30] [--store /dev/shm/pec_example]
"""

from __future__ import annotations

import argparse
import math
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def build(dev, seed: int = 0):
    import torch
    from paper_2408_04307_b200 import configs
    from paper_2408_04307_b200.arena import StateArena

    w = configs.toy()
    layout = w.layout()
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    m = layout.model
    d, ffn, L, E, V = 256, 1024, m.num_moe_layers, m.experts_per_layer, 1024

    def ne(name):
        return arena.views(f"new.{name}")["weight"]

    params = {}   # name -> (tensor view, exp_avg view, exp_avg_sq view)
    # non-expert Adam states: the ZeRO-2 flat partition [m | v] in module order
    neo = arena.views("neo.r0")["raw"].view(torch.float32)
    half = neo.numel() // 2
    flat_m, flat_v = neo[:half], neo[half:]
    pos = 0
    for name, count in m.non_expert_modules:
        p = ne(name)
        params[name] = (p, flat_m[pos:pos + count], flat_v[pos:pos + count])
        pos += count
    for layer in range(L):
        for e in range(E):
            wv = arena.views(f"ew.L{layer}.E{e}")
            ov = arena.views(f"eo.L{layer}.E{e}")
            n1 = d * ffn
            params[f"x{layer}.{e}.w1"] = (wv["w1"], ov["exp_avg"][:n1], ov["exp_avg_sq"][:n1])
            params[f"x{layer}.{e}.w2"] = (wv["w2"], ov["exp_avg"][n1:], ov["exp_avg_sq"][n1:])
    # the ZeRO flat partition is an opaque seeded blob: start its Adam
    # moments at zero.  Expert moments keep their seeded initial images
    # (exp_avg ~ N(0, 1e-3), exp_avg_sq = |N(0, 1e-6)|: valid Adam state), so
    # the "initial" recovery source (arena.fill_unit) reproduces exactly the
    # state an expert that was never saved started from.
    flat_m.zero_()
    flat_v.zero_()
    return w, layout, arena, params, dict(d=d, ffn=ffn, L=L, E=E, V=V, top_k=m.top_k)


def forward(params, shp, tokens, targets):
    """Tiny MoE LM: embed -> L x [attention-free mixer, top-2 MoE] -> tied head."""
    import torch
    import torch.nn.functional as F
    d, ffn, L, E, V, k = (shp[x] for x in ("d", "ffn", "L", "E", "V", "top_k"))

    def P(name):
        return params[name][0]

    emb = P("embed").view(V, d)
    x = emb[tokens]                                      # [T, d]
    router_ids = []
    for layer in range(L):
        ln1 = P(f"l{layer}_ln1")
        h = F.layer_norm(x, (d,), ln1[:d], ln1[d:])
        attn = P(f"l{layer}_attn").view(4, d, d)
        x = x + torch.tanh(h @ attn[0]) @ attn[3]        # mixer stand-in for attention
        ln2 = P(f"l{layer}_ln2")
        h = F.layer_norm(x, (d,), ln2[:d], ln2[d:])
        logits = h @ P(f"l{layer}_gate").view(d, E)
        weights, ids = torch.topk(torch.softmax(logits, -1), k, dim=-1)   # [T, k]
        router_ids.append(ids.reshape(-1))               # int64, counted as is
        out = torch.zeros_like(h)
        for e in range(E):
            sel = (ids == e)
            rows = sel.any(-1).nonzero(as_tuple=True)[0]
            if rows.numel() == 0:
                continue
            gate_w = (weights * sel)[rows].sum(-1, keepdim=True)
            w1 = P(f"x{layer}.{e}.w1").view(d, ffn)
            w2 = P(f"x{layer}.{e}.w2").view(ffn, d)
            out[rows] += gate_w * (F.gelu(h[rows] @ w1) @ w2)
        x = x + out
    lnf = P("lnf")
    x = F.layer_norm(x, (d,), lnf[:d], lnf[d:])
    loss = F.cross_entropy(x @ emb.t(), targets)
    return loss, torch.stack(router_ids)                 # ids [L, T*k] int64


def adam_step(params, step: int, lr=3e-3, b1=0.9, b2=0.999, eps=1e-8):
    import torch
    ps = [p for p, _, _ in params.values() if p.grad is not None]
    gs = [p.grad for p, _, _ in params.values() if p.grad is not None]
    ms = [m for p, m, _ in params.values() if p.grad is not None]
    vs = [v for p, _, v in params.values() if p.grad is not None]
    with torch.no_grad():
        torch._foreach_mul_(ms, b1)
        torch._foreach_add_(ms, gs, alpha=1 - b1)
        torch._foreach_mul_(vs, b2)
        torch._foreach_addcmul_(vs, gs, gs, value=1 - b2)
        bc1, bc2 = 1 - b1 ** step, 1 - b2 ** step
        denom = torch._foreach_sqrt(vs)
        torch._foreach_div_(denom, math.sqrt(bc2))
        torch._foreach_add_(denom, eps)
        torch._foreach_addcdiv_(ps, ms, denom, value=-lr / bc1)
    for p in ps:
        p.grad = None


def train(iters: int = 30, i_ckpt: int = 5, store_root=None, seed: int = 0, tokens: int = 512,
          on_checkpoint=None, fault_at: int = 0):
    """Returns (checkpointer, arena, losses, params).  ``on_checkpoint(buf)``
    runs after each snapshot is started (state = the snapshotted state).
    ``fault_at`` > 0 wipes the GPU state at that iteration (a lost node) and
    recovers with `PecCheckpointer.recover`: partial-expert restore from host
    memory / storage / initial images, load-aware counters reset, training
    resumes at the restart iteration (batches are a function of the
    iteration, so replayed iterations see the same data)."""
    import torch
    from paper_2408_04307_b200 import PecConfig
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore

    dev = torch.device("cuda", 0)
    torch.manual_seed(seed)
    w, layout, arena, params, shp = build(dev)
    for p, _, _ in params.values():
        p.requires_grad_(True)
    routed = tokens * shp["top_k"]
    counters = DeviceTokenCounters(shp["L"], shp["E"], dev,
                                   DeviceTokenCounters.capacity_for(1.25, [routed] * shp["L"],
                                                                    shp["E"]))
    store = DiskStore(store_root or tempfile.mkdtemp(prefix="pec_example_"))
    pec = PecConfig(k_pec=2, selection="load_aware", k_snapshot=2, k_persist=1)
    ck = PecCheckpointer(layout, arena, store, pec, "equal_pec", i_ckpt=i_ckpt, counters=counters)
    ck.prepare()                       # staging + pinned host buffers + phase tables
    g = torch.Generator(device=dev)
    losses = []
    it = 1
    while it <= iters:
        g.manual_seed(seed * 100003 + it)
        tok = torch.randint(0, shp["V"], (tokens,), device=dev, generator=g)
        tgt = tok                      # a learnable toy objective (reproduce the token)
        loss, ids = forward(params, shp, tok, tgt)
        loss.backward()
        ck.wait_pack()                 # the update may not race an in-flight pack
        adam_step(params, it)
        buf = ck.step(it, ids)         # count this iteration's routing; snapshot every i_ckpt
        if buf is not None and on_checkpoint is not None:
            on_checkpoint(buf)
        losses.append(float(loss.detach()))
        if it == fault_at:
            fault_at = 0               # one fault
            ck.finish()                # (in-flight persists land or are discarded)
            arena.buffer.zero_()       # the GPU state is gone
            out = ck.recover({0}, it)  # node 0 lost: host snapshot copies too
            for p, _, _ in params.values():
                p.grad = None
            it = out.restart_iteration + 1
            continue
        it += 1
    ck.finish()
    return ck, arena, losses, params


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--store", default=None)
    ap.add_argument("--fault-at", type=int, default=0)
    args = ap.parse_args()
    ck, arena, losses, _ = train(args.iters, store_root=args.store, fault_at=args.fault_at)
    print(f"loss {losses[0]:.3f} -> {losses[-1]:.3f}; versions {ck.engine.store.complete_versions()}")
    ck.close()


if __name__ == "__main__":
    main()
