# Round evidence on one B200: GPU suite, smoke, bench line, launch list and
# the --set full capture of the two dictionary kernels, the §8f component
# lines, then (FULL=1, default) the full-size C3/C4/C5 runs (outputs in gpurun_out/).
set -u
TAG=${TAG:-r2c}
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/${TAG}_gputest.log 2>&1
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --prof-steps 0 \
  > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k 'regex:k_hash_probe|k_verify_cells' -s 2 -c 2 -o gpurun_out/${TAG}_dict \
  python tools/one_ggr.py 2 2 > /dev/null 2>&1
timeout 600 python tools/bench_next.py > gpurun_out/${TAG}_next.jsonl 2> gpurun_out/${TAG}_next.err
echo done
[ "${FULL:-1}" = 1 ] || exit 0
for c in 3 4 5; do
  timeout 700 python tools/full_size.py $c --paths=device --reps=3 >> gpurun_out/${TAG}_full.jsonl 2>> gpurun_out/${TAG}_full.err
done
