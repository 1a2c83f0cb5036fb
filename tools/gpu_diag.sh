for a in 0 8 0 8; do echo -n "bwd_ablate=$a "; DKV_BWD_ABLATE=$a REPS=80 timeout 200 python tools/power_probe.py bwd; done
