for mf in 2; do
for it in 640 1920; do
  PDLP_OPTS="{\"step_safety\": 0.9, \"matrix_free\": $mf}" torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + it % 97 + mf)) \
      tools/c4_solve.py 32 2024 slowest 1e-12 $it 0 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($mf, d['iters'], d['device_seconds_max'])"
done
done
