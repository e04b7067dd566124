cd /root/repo
cp paper_2605_02568_b200/lib/libcsaidx_cuda.so /tmp/lib_new.so
for r in 1 2 3; do
for v in new old; do
  if [ $v = old ]; then cp scripts/_av_old/libcsaidx_cuda.so paper_2605_02568_b200/lib/libcsaidx_cuda.so; else cp /tmp/lib_new.so paper_2605_02568_b200/lib/libcsaidx_cuda.so; fi
  a=$(timeout 120 python scripts/bench_attention.py 8192 65536 1024 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_launch'],3))")
  b=$(timeout 120 python scripts/bench_attention.py 2048 65536 2048 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_launch'],3))")
  echo $v $a $b
done
done
cp /tmp/lib_new.so paper_2605_02568_b200/lib/libcsaidx_cuda.so
