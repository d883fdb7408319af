run() { tag=$1; shift; env "$@" timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/r02_sweep_$tag.json 2> gpurun_out/r02_sweep_$tag.err; }
EXTRA="--collectives nccl" run nccl_default X=1
EXTRA="--collectives nccl" run nccl_max4 OSH_NCCL_MAX_CTAS=4
EXTRA="--collectives nccl" run nccl_max8 OSH_NCCL_MAX_CTAS=8
EXTRA="--collectives nccl" run nccl_pol1 OSH_NCCL_CTA_POLICY=1
EXTRA="--collectives nccl" run nccl_pol2 OSH_NCCL_CTA_POLICY=2
EXTRA="--tp 2" run tp2_default X=1
EXTRA="--tp 2" run tp2_max8 OSH_NCCL_MAX_CTAS=8
EXTRA="--tp 2" run tp2_pol2 OSH_NCCL_CTA_POLICY=2
