# scratch: final 1-GPU checks + profile round
O=gpurun_out/final2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo rc=$? >> $O/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
OUT=$O/prof bash tools/profile_round.sh > $O/prof.log 2>&1
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
