set -x
python bench.py --steps 200 --warmup 10 > gpurun_out/r02_bench_b200.json 2> gpurun_out/r02_bench_b200.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/r02_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ringp -s 30 -c 1 -o gpurun_out/r02_ring256 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-configs --no-extra-formats > gpurun_out/r02_ncu_ring.log 2>&1
ls -la gpurun_out
