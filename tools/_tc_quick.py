import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1510_06706_b200 import Context, ops
from oracle import oracle as O
ctx = Context(0)
rng = np.random.default_rng(0)
def t(a): return torch.as_tensor(np.ascontiguousarray(a), device='cuda')
for (B, fi, fo, n, k, s) in [(1, 16, 16, (6,6,6), (1,1,1), (1,1,1)), (2, 3, 40, (9,8,10), (3,3,3), (1,1,1)), (1, 40, 120, (12,12,12), (5,5,5), (2,2,2)), (1, 120, 120, (11,11,11), (5,5,5), (2,2,2))]:
    x = rng.uniform(0,1,size=(B,fi)+n).astype(np.float32)
    w = rng.uniform(-0.1,0.1,size=(fo,fi)+k).astype(np.float32)
    y = ops.conv_fwd(ctx, t(x), t(w), k, s, act='none', engine='direct').cpu().numpy()
    err = max(O.max_rel_error(y[b,o], sum(O.conv_valid(x[b,i], w[o,i], s) for i in range(fi))) for b in range(B) for o in range(min(fo,8)))
    print('fwd', (B,fi,fo,n,k,s), 'err', err, flush=True)
    m = y.shape[2:]
    g = rng.uniform(-1,1,size=(B,fo)+m).astype(np.float32)
    if fi >= 16:
        dx = ops.conv_dgrad(ctx, t(g), t(w), k, s, engine='direct').cpu().numpy()
        err = max(O.max_rel_error(dx[b,i], sum(O.conv_full(g[b,o], O.reflect(w[o,i]), s) for o in range(fo))) for b in range(B) for i in range(min(fi,8)))
        print('dgrad err', err, flush=True)
    dw = ops.conv_wgrad(ctx, t(x), t(g), k, s, engine='direct').cpu().numpy()
    err = max(O.max_rel_error(dw[o,i], sum(O.kernel_grad(x[b,i], g[b,o], k, s) for b in range(B))) for o in range(min(fo,6)) for i in range(min(fi,6)))
    print('wgrad err', err, flush=True)
# big wgrad accuracy (long K)
B, fi, fo, n, k, s = 2, 8, 16, (40,40,40), (3,3,3), (1,1,1)
x = rng.uniform(0,1,size=(B,fi)+n).astype(np.float32); m=(38,38,38)
g = rng.uniform(-1,1,size=(B,fo)+m).astype(np.float32)
dw = ops.conv_wgrad(ctx, t(x), t(g), k, s, engine='direct').cpu().numpy()
err = max(O.max_rel_error(dw[o,i], sum(O.kernel_grad(x[b,i], g[b,o], k, s) for b in range(B))) for o in range(3) for i in range(3))
print('wgrad long-K err', err, 'max |dw|', np.abs(dw).max(), flush=True)
def bench(fn, reps=3):
    fn(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/reps
for (B, fi, fo, n, k, s) in [(1, 120, 120, (90,90,90), (5,5,5), (2,2,2)), (2, 120, 120, (80,80,80), (5,5,5), (4,4,4)), (8, 40, 40, (42,42,42), (3,3,3), (1,1,1)), (1, 1, 120, (95,95,95), (5,5,5), (1,1,1)), (1, 80, 80, (62,62,62), (7,7,7), (2,2,2))]:
    x = torch.rand((B,fi)+n, device='cuda'); w = (torch.rand((fo,fi)+k, device='cuda')-0.5)*0.01
    m=[n[a]-s[a]*(k[a]-1) for a in range(3)]
    g = torch.rand((B,fo)+tuple(m), device='cuda')-0.5
    fl = 2*B*fi*fo*np.prod(m)*np.prod(k)
    for eng in ['direct', 'simt']:
        tf = bench(lambda: ops.conv_fwd(ctx, x, w, k, s, act='relu', engine=eng))
        td = bench(lambda: ops.conv_dgrad(ctx, g, w, k, s, engine=eng)) if fi >= 16 else float('nan')
        tw = bench(lambda: ops.conv_wgrad(ctx, x, g, k, s, engine=eng))
        print(eng, (B,fi,fo,n,k,s), f'fwd {tf*1e3:.2f} ms {fl/tf/1e12:.1f} | dgrad {td*1e3:.2f} ms {fl/td/1e12:.1f} | wgrad {tw*1e3:.2f} ms {fl/tw/1e12:.1f} TFLOP/s', flush=True)
