# session 5: k_stage3 with lane-replicated antilog lookups (HQC_S3_REPL=1 build, scripts/libx_s3repl.so) vs the default
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
# parity of the variant: the stage-3 test file's cases through the variant library, then a soak at HQC-5
timeout 600 python - > gpurun_out/s3repl_parity.log 2>&1 <<'PY'
import sys, os
sys.path.insert(0, "tests"); sys.path.insert(0, "scripts")
from paper_2512_12904_b200 import hqc
hqc.LIB_PATH = os.path.abspath("scripts/libx_s3repl.so")
import numpy as np, torch, oracle
for level in (1, 3, 5):
    p = oracle.params(level)
    rng = np.random.default_rng(level)
    B = 3000
    msg = rng.integers(0, 256, (B, p.k), dtype=np.uint8)
    sym = np.stack([oracle.rs_encode(m, p.n1, p.k) for m in msg])
    for i in range(B):
        kind = i % 4
        ne = 0 if kind == 0 else int(rng.integers(1, p.delta + 1)) if kind == 1 else int(rng.integers(p.delta + 1, 2 * p.delta + 1)) if kind == 2 else -1
        if ne < 0:
            sym[i] = rng.integers(0, 256, p.n1, dtype=np.uint8)
        elif ne:
            pos = rng.choice(p.n1, ne, replace=False)
            sym[i, pos] ^= rng.integers(1, 256, ne, dtype=np.uint8)
    ref, ok_ref = oracle.rs_decode_batch(p, sym)
    d = torch.from_numpy(sym).cuda()
    m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda"); ok = torch.empty(B, dtype=torch.uint8, device="cuda")
    hqc.hqc_rs_decode_batch(level, d, m, ok); torch.cuda.synchronize()
    got = m.cpu().numpy().reshape(B, p.k)
    print(level, "rs rows differ:", int((got != ref).any(axis=1).sum()), "ok differ:", int((ok.cpu().numpy() != np.asarray(ok_ref).astype(np.uint8)).sum()), flush=True)
import soak_parity
sys.argv = ["soak", "2", "5"]
soak_parity.main()
PY
echo "parity exit $?" >> gpurun_out/s3repl_parity.log
timeout 600 python scripts/exp_lib_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libx_s3repl.so 5:32768,5:65536,5:262144,5:1048576 > gpurun_out/ab_s3repl.log 2>&1
