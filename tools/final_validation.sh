# round-end validation on one B200: GPU suite, smoke, default bench, reference arm, launch list
timeout 2900 python -m pytest tests -m gpu -q > gpurun_out/final_gpu.log 2>&1; tail -2 gpurun_out/final_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 3 --leapfrogs 5 --e2e-steps 1 --no-cpu-baseline > gpurun_out/final_ncu.log 2>&1; echo ncu rc=$?
