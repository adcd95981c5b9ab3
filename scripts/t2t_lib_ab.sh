mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
echo old; STL_LIB=$PWD/scripts/ab/lib_old.so python scripts/bench_t2t.py --steps 10 | cut -c100-200
echo new; python scripts/bench_t2t.py --steps 10 | cut -c100-200
done
python scripts/profile_t2t.py 2>/dev/null | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_total'], d['families_ms'])"
timeout 300 python scripts/transform_probe.py | tail -1 | cut -c1-250
} > gpurun_out/t2t_lib_ab.log 2>&1
cat gpurun_out/t2t_lib_ab.log
