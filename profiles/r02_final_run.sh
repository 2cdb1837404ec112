set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/ncu_list.log 2>&1; echo list rc $?
ncu --set full --clock-control none --import-source on -k regex:ringp -s 30 -c 1 -f -o gpurun_out/ring256 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-configs --no-extra-formats > gpurun_out/ncu_full.log 2>&1; echo full rc $?
ncu --set full --clock-control none --import-source on -k regex:ringp -s 8 -c 1 -f -o gpurun_out/ring512 python tests/ring_probe.py 512 > gpurun_out/ncu_full512.log 2>&1; echo full512 rc $?
ls -la gpurun_out
