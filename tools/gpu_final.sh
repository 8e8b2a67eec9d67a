# Round-end evidence at HEAD: GPU tests, smoke, the round-2 profile set (bench lines, launch lists,
# K1 captures, drift), the post-K1 ncu summary at k = 2^20
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo gputest_rc=$?; tail -3 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -2 $O/smoke.log
bash tools/profile_r2.sh $O > $O/profile.log 2>&1; echo profile_rc=$?
python tools/bench_summary.py $O/bench_full.json
cat $O/bench_ref.json | head -c 600; echo
bash tools/prof_tail.sh $O 1048576 uniform
rm -f $O/*.ncu-rep
du -sh $O
