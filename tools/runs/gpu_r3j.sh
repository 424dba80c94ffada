#!/bin/bash
# configs[4] (Llama-2-70B shape, head-sharded) at 16 layers: TP=1, and TP=2 as two processes sharing GPU 0
OUT=gpurun_out/r3j
mkdir -p $OUT
timeout 900 python bench.py --config c5 --c5-layers 16 --c5-modules 16 --steps 5 --warmup 3 > $OUT/c5_tp1.json 2> $OUT/c5_tp1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --config c5 --c5-layers 16 --c5-modules 16 --share-device --steps 5 --warmup 3 > $OUT/c5_tp2_shared.json 2> $OUT/c5_tp2_shared.err
