# numpy (pageable) host path: exactness tests, then e2e timings by copy-thread count
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_q2.py -m gpu -x -q -k "pageable or pinned or q2_operator" > gpurun_out/pg_tests.log 2>&1; echo "tests rc=$?"
cat > /tmp/pg.py <<'PY'
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1902_08112_b200 import configs, model
from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
for cfg in sys.argv[1:]:
    prob = configs.make(cfg)
    mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
    op = PhaseFieldOperator(prob.disc.finest, prob.state, ConstraintMask(mask.is_constrained, mask.inhomogeneity),
                            prob.params, SplitKind.NOSPLIT)
    v = prob.v.copy()
    out = np.empty_like(v)
    def med(fn, reps=15):
        for _ in range(3): fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
        return np.median(ts) * 1e3
    model.PAGEABLE_PIPELINE = False
    a = med(lambda: op.apply(v))
    model.PAGEABLE_PIPELINE = True
    b = med(lambda: op.apply(v))
    c = med(lambda: op.apply(v, out=out))
    hv = torch.from_numpy(v).pin_memory(); ho = torch.empty_like(hv).pin_memory()
    d = med(lambda: op.apply(hv, out=ho))
    print(f"== {cfg} threads={os.environ.get('PFFMG_COPY_THREADS','default')} n={v.size}: plain {a:.3f} ms  pageable {b:.3f} ms  pageable(out=) {c:.3f} ms  pinned {d:.3f} ms", flush=True)
PY
for t in 1 2 4 6 8 12 16; do PFFMG_COPY_THREADS=$t python /tmp/pg.py cfg2; done
python /tmp/pg.py cfg2 cfg3 cfg4
