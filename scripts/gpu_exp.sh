cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/par.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle
from paper_2512_12904_b200 import hqc
hqc.LIB_PATH = os.path.abspath(sys.argv[1])
from workloads import valid_batch, adversarial_batch
for level in (3,):
    for W in (valid_batch(level, 40000, 300), ):
        p = hqc.params(level)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()
        B = W["u"].shape[0]
        m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
        hqc.hqc_decrypt_batch(level, d(W["u"]), d(W["v"]), d(W["y"]), m)
        torch.cuda.synchronize()
        ref = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
        print("parity", (m.cpu().numpy().reshape(B, p.k) == ref).all())
PY
for f in scripts/libx_*.so; do python /tmp/par.py $f >> gpurun_out/exp.log 2>&1; done
for r in 1 2; do for f in scripts/libx_*.so; do timeout 120 python scripts/time_lib.py $f 3 >> gpurun_out/exp.log 2>&1; done; done
