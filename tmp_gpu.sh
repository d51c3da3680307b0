cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 400 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_c2_ref.json 2> gpurun_out/bench_c2_ref.err
