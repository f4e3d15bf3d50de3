set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r02c_bench_wan.json 2> gpurun_out/r02c_bench_wan.err
python bench.py --workload cogvideox --no-cpu-baseline > gpurun_out/r02c_bench_cogvideox.json 2> gpurun_out/r02c_bench_cog.err
python bench.py --workload hunyuan --steps 10 --no-cpu-baseline --sp-sim 0 > gpurun_out/r02c_bench_hunyuan.json 2> gpurun_out/r02c_bench_hun.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02c_bench_wan_reference.json 2> gpurun_out/r02c_ref.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sparse_attn -s 3 -c 1 -o gpurun_out/r02c_cog_full python bench.py --workload cogvideox --steps 1 --warmup 3 --no-cpu-baseline --sp-sim 0 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sparse_attn -s 3 -c 1 -o gpurun_out/r02c_wan_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sp-sim 0 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_wan.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --sp-sim 0 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
