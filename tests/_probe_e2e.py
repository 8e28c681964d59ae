# Diagnostics: what bounds the end-to-end loop (host issue rate, PCIe copies, the chain)?
import sys, time
import torch
sys.path.insert(0, '.')
import bench
from paper_2512_12949_b200 import runtime

dev = torch.device('cuda', 0)
name = 'llama1b'
kind, act, m, n, k, l, _ = bench.WORKLOADS[name]
graph = bench.graph_of(name)
t = bench.make_device_inputs(kind, m, n, k, l, seed=1, device=dev)
cfg = runtime.lower(graph, None, 148, 'pair')
out = torch.empty((m, l), dtype=torch.bfloat16, device=dev)
host_a = t['A'].cpu().pin_memory()
host_e = torch.empty((m, l), dtype=torch.bfloat16).pin_memory()
s = torch.cuda.current_stream()
N = 200

def timed(fn):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0 = time.perf_counter(); a.record()
    for _ in range(N): fn()
    b.record(); c1 = time.perf_counter(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / N, (c1 - c0) * 1e6 / N

print('launch only          gpu %.1f us/step  host issue %.1f us/step' % timed(lambda: runtime.launch(graph, cfg, t, out=out)))
s0 = torch.cuda.Stream()
def h2d_created():
    with torch.cuda.stream(s0): t['A'].copy_(host_a, non_blocking=True)
print('H2D on created stream gpu %.1f us/step  host issue %.1f us/step' % timed(h2d_created))
print('H2D 2 MiB only       gpu %.1f us/step  host issue %.1f us/step' % timed(lambda: t['A'].copy_(host_a, non_blocking=True)))
print('D2H 2 MiB only       gpu %.1f us/step  host issue %.1f us/step' % timed(lambda: host_e.copy_(out, non_blocking=True)))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): t['A'].copy_(host_a, non_blocking=True)
    with torch.cuda.stream(s2): host_e.copy_(out, non_blocking=True)
print('H2D || D2H           gpu %.1f us/step  host issue %.1f us/step' % timed(both))
ev = [torch.cuda.Event() for _ in range(4)]
print('event create+record  gpu %.1f us/step  host issue %.1f us/step' % timed(lambda: torch.cuda.Event().record()))
for steps in (200,):
    r = bench.e2e_pipelined(graph, cfg, t, host_a, kind, m, l, steps, dev)
    print('pipelined e2e        gpu %.1f us/step' % (r['ms_total'] * 1e3 / steps))

# variants of the pipelined loop
sets = [dict((kk, v.clone()) for kk, v in t.items() if kk != 'A') for _ in range(4)]
devs_a = [torch.empty_like(t['A']) for _ in range(2)]
outs = [torch.empty((m, l), dtype=torch.bfloat16, device=dev) for _ in range(2)]
hosts_e = [torch.empty((m, l), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
hosts_a = [host_a, host_a.clone().pin_memory()]
sc, si, so = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def loop(n, h2d, ker, d2h, rotate=True):
    kd = [torch.cuda.Event() for _ in range(n)]; od = [torch.cuda.Event() for _ in range(n)]; ai = [torch.cuda.Event() for _ in range(n)]
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record(sc); si.wait_event(st); so.wait_event(st)
    c0 = time.perf_counter()
    for i in range(n):
        b = i & 1
        if h2d:
            if i >= 2: si.wait_event(kd[i - 2])
            with torch.cuda.stream(si): devs_a[b].copy_(hosts_a[b], non_blocking=True)
            ai[i].record(si); sc.wait_event(ai[i])
        if i >= 2 and d2h: sc.wait_event(od[i - 2])
        if ker: runtime.launch(graph, cfg, dict(sets[i % 4] if rotate else sets[0], A=devs_a[b]), out=outs[b], stream=sc)
        kd[i].record(sc)
        if d2h:
            so.wait_event(kd[i])
            with torch.cuda.stream(so): hosts_e[b].copy_(outs[b], non_blocking=True)
            od[i].record(so)
    if d2h: sc.wait_event(od[n - 1])
    en.record(sc); c1 = time.perf_counter(); torch.cuda.synchronize()
    return st.elapsed_time(en) * 1e3 / n, (c1 - c0) * 1e6 / n
for args in [(1, 1, 1), (0, 1, 0), (1, 0, 0), (0, 0, 1), (1, 0, 1), (1, 1, 0), (0, 1, 1)]:
    loop(4, *args)
    print('h2d %d kernel %d d2h %d: gpu %.1f us/step host %.1f us/step' % (args + loop(200, *args)))
print('no rotation (1,1,1): gpu %.1f us/step host %.1f' % loop(200, 1, 1, 1, rotate=False))

def h2d_variant(n, alt_host, alt_dev, stream_kind):
    ss = {'legacy': torch.cuda.default_stream(), 'created': si, 'hiprio': torch.cuda.Stream(priority=-1)}[stream_kind]
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); st.record(sc); ss.wait_event(st)
    for i in range(n):
        b = i & 1
        with torch.cuda.stream(ss):
            devs_a[b if alt_dev else 0].copy_(hosts_a[b if alt_host else 0], non_blocking=True)
    e = torch.cuda.Event(); e.record(ss); sc.wait_event(e)
    en.record(sc); torch.cuda.synchronize()
    return st.elapsed_time(en) * 1e3 / n
for v in [(0, 0, 'legacy'), (1, 1, 'legacy'), (0, 0, 'created'), (1, 1, 'created'), (0, 0, 'hiprio')]:
    h2d_variant(4, *v)
    print('H2D alt_host %d alt_dev %d stream %s: %.1f us/step' % (v + (h2d_variant(200, *v),)), flush=True)
