# A/B timing of alternative in-tree builds (DKV_LIB) on one box: C3 two-call backward
LIBS=${LIBS:-"libdkv.so libdkv_old.so"}
for L in $LIBS; do DKV_LIB=$L timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/$L parity: /"; done
for i in 1 2; do
for L in $LIBS; do echo -n "$L "; DKV_LIB=$L timeout 200 python tools/ablate_bwd.py 0; done
done
