# Single-GPU per-iteration A/B of library variants on the 16-chassis LP (fixed iterations)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29544"
for v in default ${LIBS:-c1}; do
  for it in 320 640; do
    if [ $v = default ]; then L=""; else L="TECCL_B200_LIB=build_variants/libteccl_$v.so"; fi
    env $L timeout 600 $R tools/dist_run.py 16 1 3860 1e-12 0 $it 2>gpurun_out/big_$v.err | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['iters'], round(d['device_seconds_max'],3))"
  done
done
