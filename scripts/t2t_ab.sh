mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_t2t_vit.py tests/test_training.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for i in 1 2; do
python scripts/bench_t2t.py --steps 10
python scripts/bench_t2t.py --steps 10 --no-fused-tokens
done
python scripts/bench_t2t.py --steps 10 --dense
python scripts/profile_t2t.py 2>/dev/null | head -1 | cut -c1-1500
} > gpurun_out/t2t_ab.log 2>&1
cat gpurun_out/t2t_ab.log
