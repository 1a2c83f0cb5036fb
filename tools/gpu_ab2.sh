timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 2>&1 | tail -5
for i in 1 2; do
for L in libdkv.so libdkv_old.so; do echo $L; DKV_LIB=$L timeout 200 python tools/ablate_bwd.py 0; done
done
