cd "${GRAFT_REPO_ROOT}"
O=gpurun_out/r2a; mkdir -p $O
bash tools/box_probe.sh > $O/probe.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
