L=paper_2603_10026_b200
cp $L/librf_cuda.so $L/librf_cuda_new.so
run() { timeout 300 python bench.py --config $2 --also "" --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 cfg$2', d['value'], 'e2e', d['e2e']['value'])"; }
for c in 1 3 0; do
  cp $L/librf_cuda_new.so $L/librf_cuda.so; run new $c
  cp $L/librf_cuda_old.so $L/librf_cuda.so; run old $c
done
cp $L/librf_cuda_new.so $L/librf_cuda.so
