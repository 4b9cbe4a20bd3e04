cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_batch or striding or decrypt_valid or variants or adversarial_quarters or edges" > gpurun_out/pytest_sb.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sb.log
timeout 600 python scripts/exp_sb_phases.py run > gpurun_out/sb_phases.log 2>&1
timeout 900 python scripts/sweep_launch.py small > gpurun_out/sweep_small.log 2>&1
