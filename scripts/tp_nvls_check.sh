#!/bin/bash
# 4-GPU box: the TP multi-GPU tests, then DP2xTP2 bench lines on NVLS (auto)
# and NCCL, and DP4 NVLS for the same-box comparison. Output: gpurun_out/tpn/
mkdir -p gpurun_out/tpn
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests/test_gpu_multi.py -q -rA -k "tp2" > gpurun_out/tpn/tests.log 2>&1
  echo "tests rc=$?" >> gpurun_out/tpn/tests.log
fi
bench() {  # name, args
  local name=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 4 \
    --steps 10 --warmup 3 --no-cpu-baseline "$@" \
    > gpurun_out/tpn/$name.json 2> gpurun_out/tpn/$name.err
  echo "$name rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/tpn/$name.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('phases_ms_rank0'), d['max_mean_rank_load'].get('per_rank_compute_ms'), d['e2e']['value'] if d.get('e2e') else None, d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
}
for name in ${BENCHES:-tp2_auto dp4_auto tp2_nccl}; do
  case $name in
    tp2_auto) bench tp2_auto --tp 2 ;;
    tp2_nccl) bench tp2_nccl --tp 2 --collectives nccl ;;
    dp4_auto) bench dp4_auto ;;
    tp2_seqov) OSH_SEQ_OVERLAP=1 bench tp2_seqov --tp 2 ;;
  esac
done
