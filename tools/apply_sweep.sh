for thr in 128 96 64; do
echo "thr=$thr $(RBF_APPLY_SYM_THREADS=$thr timeout 200 python tools/apply_bench.py c4 2>&1 | tail -1)"
done
