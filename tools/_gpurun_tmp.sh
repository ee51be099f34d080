python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "reference_api or gamma or multirank or cfg3_scale" > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/gputest.log; cat gpurun_out/bench.json; cat gpurun_out/bench_ref.json; tail -5 gpurun_out/bench.err
