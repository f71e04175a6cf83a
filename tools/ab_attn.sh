# A/B of two librf_cuda builds on one box (same session): the in-tree
# librf_cuda.so ("new") vs paper_2603_10026_b200/librf_cuda_old.so ("old").
#   bash tools/ab_attn.sh [config index] [repeats] [steps]
cfg=${1:-1}; rep=${2:-2}; steps=${3:-20}
L=paper_2603_10026_b200
cp $L/librf_cuda.so $L/librf_cuda_new.so
run() { timeout 300 python bench.py --config $cfg --also "" --steps $steps --warmup 5 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for r in $(seq $rep); do
  cp $L/librf_cuda_new.so $L/librf_cuda.so; run new
  cp $L/librf_cuda_old.so $L/librf_cuda.so; run old
done
cp $L/librf_cuda_new.so $L/librf_cuda.so
