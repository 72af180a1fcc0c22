#!/bin/bash
# A/B of the per-half group barriers (tc_pass.cuh hsync) and the encoder's vector-bit-7 choice,
# then the parity suites that cover the tensor-core pass.
cd "${GRAFT_REPO_ROOT:-.}"
O=${1:-gpurun_out/ab_hs}
mkdir -p $O
bash tools/ab_env.sh "c2" "c2 STV_NO_HALFSYNC=1" "c2 STV_NO_HALFSYNC=1 STV_NO_V7CHAIN=1" "c2" \
  "c3" "c3 STV_NO_HALFSYNC=1 STV_NO_V7CHAIN=1" "c4" "c4 STV_NO_HALFSYNC=1 STV_NO_V7CHAIN=1" > $O/ab.txt 2>&1
cat $O/ab.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py tests/test_gpu_fullsize.py -m gpu -x -q \
  -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
