for i in 1 2; do
for lib in build/oldsplit/libbf16x.so paper_1904_06376_b200/libbf16x.so build/plainst/libbf16x.so; do
BF16X_LIB=$lib python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['split_gbs']), round(d['secondary']['value'],1), round(d['secondary']['ms_per_step']*1e3,1), round(d['secondary']['split_gbs']))"
done; done
