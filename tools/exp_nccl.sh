R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 1000 --precision bf16 --replay 100000 --e2e-steps 20"
S='import json,sys
for l in sys.stdin:
  if l.startswith("{"): d=json.loads(l); print(d["value"], d["ms_per_step"], d["regions_us"])'
echo default; $R 2>/dev/null | python -c "$S"
echo LL; NCCL_PROTO=LL $R 2>/dev/null | python -c "$S"
echo LL128; NCCL_PROTO=LL128 $R 2>/dev/null | python -c "$S"
echo NVLS; NCCL_ALGO=NVLS $R 2>/dev/null | python -c "$S"
echo RING_LL; NCCL_ALGO=Ring NCCL_PROTO=LL $R 2>/dev/null | python -c "$S"
