"""Warp/scheduler replay of k_qp_admm scheduling from dumped per-instance iteration counts
(tools/qp_iters_dump.py): python tools/admm_sched_model.py BATCH.  Model, not a measurement:
per batch step a scheduler takes (active warps)/3 of a full-contention step."""
import numpy as np, sys
it = np.load('/root/repo/gpurun_out/qp_iters_cfg3.npy').astype(np.int64)
n = it.size; S = 148*4; W = S*3; B = int(sys.argv[1])
sched = np.arange(W) % S
def steptime(busy):
    c = np.bincount(sched[busy], minlength=S) if busy.any() else np.zeros(S)
    return c.max()/3
def run(T, p2=True):
    rem = np.zeros((W,32), np.int64); nxt = 0; t = 0.; spilled = []; live = np.ones(W, bool); ex=False
    while True:
        need = (rem == 0) & live[:,None]
        if nxt < n:
            idx = np.flatnonzero(need.ravel())[: n - nxt]
            rem.ravel()[idx] = it[nxt:nxt+idx.size]; nxt += idx.size
        else:
            ex = True
        act = (rem > 0).sum(1)
        if ex and T > 0:
            sp = live & (act <= T) & (act > 0)
            for w in np.flatnonzero(sp): spilled.extend(rem[w][rem[w] > 0].tolist()); rem[w] = 0
            live &= ~sp
        busy = (rem > 0).any(1)
        if not busy.any(): break
        t += steptime(busy); rem = np.maximum(rem - B, 0)
    t1 = t
    if spilled:
        r = np.array(spilled); k = -(-r.size // 32); r = np.concatenate([r, np.zeros(k*32 - r.size, int)]).reshape(k, 32)
        # pass-2 warps placed round-robin over schedulers (persistent: assume all resident if k <= W)
        s2 = np.arange(k) % S
        t += 0.5  # launch + state reload overhead (~half a step)
        while (r > 0).any():
            busy = (r > 0).any(1)
            c = np.bincount(s2[busy], minlength=S); t += max(c.max(), 1)/3 if c.max() < 3 else c.max()/3
            r = np.maximum(r - B, 0)
    return t1, t, len(spilled)
base = run(0)[1]
print('baseline time', base, 'ideal', it.sum()/32/B/W)
for T in (4, 8, 12, 16, 20, 24):
    t1, t, ns = run(T); print('T', T, 'pass1', round(t1,1), 'total', round(t,1), 'spilled', ns, 'gain %', round(100*(1-t/base),2))
it0 = it.copy()
it = np.sort(it0)[::-1].copy(); print('LPT oracle', run(0)[1])
st = np.load('/root/repo/gpurun_out/qp_status_cfg3.npy'); print('status counts', np.bincount(st))
# correlation of iterations with position (edge order)?
print('mean iters by decile of instance index', [int(x.mean()) for x in np.array_split(it0, 10)])
