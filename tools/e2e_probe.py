"""Phase breakdown of bench.py's e2e path (host FieldSet -> load -> K x step() -> state())."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1309_1230_b200 import ExecutorKind, Stepper
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc, _ = bench.scenario_for(cfg, 1)
spec = sc.spec
pinned = [torch.empty((spec.ny, spec.nx), dtype=torch.float64).pin_memory() for _ in range(4)]
src = sc.build()
for tns, a in zip(pinned, (src.z, src.h, src.qx, src.qy)):
    tns.numpy()[:] = a
outs = [torch.empty((spec.ny, spec.nx), dtype=torch.float64).pin_memory() for _ in range(3)]
for rep in range(2):
    st = Stepper(spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=False))
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    st.load_rows(*[p.numpy() for p in pinned], t=0.0); t.append(time.perf_counter())
    dt = st.compute_dt(math.inf); t.append(time.perf_counter())
    for k in range(steps):
        dt = st.step(dt, k).dt_next
    t.append(time.perf_counter())
    st.state_rows(*[o.numpy() for o in outs]); t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"rep {rep}: load {d[0]:.1f} ms, compute_dt {d[1]:.1f} ms, {steps} steps {d[2]:.1f} ms "
          f"({d[2]/steps:.3f}/step), state {d[3]:.1f} ms, total {sum(d):.1f} ms")
    st.close()
