#!/bin/bash
# Functional test of bench.py's N > 1 path on a one-GPU box (never a timing): torchrun ranks on cuda:0 over
# gloo (host-staged exchanges). c4 at 2 and 4 ranks (Gram blocks exchanged, 1/N of X uploaded per rank),
# c2 at 8 ranks (k = 5 < 8: replicated blocks, ranks without folds join only the curve exchange).
o=gpurun_out
export RP_BENCH_BACKEND=gloo RP_BENCH_SAME_DEVICE=1
for spec in "c4 2" "c4 4" "c2 8"; do
  set -- $spec
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 \
      --master-port $((29500 + $2)) bench.py --gpus $2 --steps 2 --warmup 3 --config $1 \
      > $o/ranks_$1_n$2.json 2> $o/ranks_$1_n$2.err
  echo "$1 N=$2 rc=$?"; tail -c 400 $o/ranks_$1_n$2.json; echo; tail -3 $o/ranks_$1_n$2.err
done
