# functional check of the N > 1 bench paths on a one-GPU box (gloo; both ranks on GPU 0)
export SGP_DIST_BACKEND=gloo
for w in c2 c5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --workload $w --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "$w rc=$? lines=$(wc -l < gpurun_out/mr_$w.json)"; head -c 300 gpurun_out/mr_$w.json; echo
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 1 --warmup 1 --leapfrogs 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/mr_c4.json 2> gpurun_out/mr_c4.err
echo "c4 rc=$? lines=$(wc -l < gpurun_out/mr_c4.json)"; head -c 300 gpurun_out/mr_c4.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "ref rc=$? lines=$(wc -l < gpurun_out/mr_ref.json)"
