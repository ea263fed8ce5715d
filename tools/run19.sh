for p in 64 80 96; do echo "panel SMs $p"; MP_PANEL_SMS=$p timeout 300 python tools/probe_scaling.py 16384 --noprof 2>&1; done
MP_PANEL_SMS=64 timeout 300 python tools/probe_scaling.py 4096 8192 --noprof 2>&1
