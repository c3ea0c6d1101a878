# scratch A/B script for gpurun (edited per experiment)
O=gpurun_out/full2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo rc=$? >> $O/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --circuit hea > $O/bench_hea.json 2> $O/bench_hea.err
