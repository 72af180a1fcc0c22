cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -k "c4 or c3" -m gpu -q -s -p no:cacheprovider 2>&1 | grep -E "PARITY|passed|failed|Error"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | cut -c1-400
