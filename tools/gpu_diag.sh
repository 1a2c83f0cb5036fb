for a in 0 4 0 4; do echo -n "fwd_ablate=$a "; DKV_FWD_ABLATE=$a REPS=250 timeout 200 python tools/power_probe.py fwd; done
