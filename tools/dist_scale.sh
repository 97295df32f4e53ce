#!/bin/bash
# Strong scaling of one row-partitioned LP: N = 1, 2, 4 (and 8 if present).
# usage: tools/dist_scale.sh CHASSIS CHUNKS K EPS MAXGPUS
C=$1; CH=$2; K=$3; EPS=$4; MAXG=${5:-4}; ITERS=${6:-5000000}
port=29600
for n in 1 2 4 8; do
  [ $n -gt $MAXG ] && break
  port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port tools/dist_run.py $C $CH $K $EPS 0 $ITERS 2>&1 | grep '^{'
done
