mkdir -p gpurun_out
for wl in wan cogvideox hunyuan; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_fwd -s 3 -c 1 -o gpurun_out/r02b_${wl}_full python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --sp-sim 0 > gpurun_out/r02b_ncu_$wl.log 2>&1; echo "$wl ncu rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_wan.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sp-sim 0 > /dev/null 2>&1; echo "launches rc=$?"
