python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc $?
python -c "import __graft_entry__ as g; g.smoke()"
