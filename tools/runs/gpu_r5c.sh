#!/bin/bash
# multi-process data path on one GPU: the multiproc GPU tests and the DP bench as two ranks sharing GPU 0
OUT=gpurun_out/r5c
mkdir -p $OUT
timeout 1300 python -m pytest tests/test_gpu_multiproc.py -m gpu -q -p no:cacheprovider -rs > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 900 python bench.py --gpus 2 --share-device --steps 5 --warmup 3 --skip-cpu --skip-slow --skip-c3 --skip-sweep \
  --micro-batches 32 > $OUT/bench_dp2_share.json 2> $OUT/bench_dp2_share.err; echo rc=$? >> $OUT/bench_dp2_share.err
