mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/s_gputests.log
timeout 900 python bench.py > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --workload cogvideox --sp-sim 0 > gpurun_out/s_bench_cog.json 2> gpurun_out/s_bench_cog.err; echo "bench cog rc=$?"
