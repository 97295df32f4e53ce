# Row-partitioned solves on NG GPUs: fused halo (default) vs separate halo kernels.
# Line 1: configs[1] to 1e-4 with the single-GPU comparison; line 2: 4-chassis
# K=800 for a fixed 6400 iterations (per-iteration time).
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1 --master-port 29533"
for f in ${FUSED:-1 2 0}; do
  PDLP_OPTS="{\"fused_halo\": $f}" timeout 300 $R tools/dist_run.py 2 2 530 1e-4 1 2>&1 | grep '^{' | tail -1
  PDLP_OPTS="{\"fused_halo\": $f}" timeout 300 $R tools/dist_run.py 4 1 800 1e-12 0 6400 2>&1 | grep '^{' | tail -1
done
