PROBE_VARIANTS=w2,w3,w4 timeout 300 python tools/tc_probe.py c2 2>&1 | grep shape
ESOM_TC2_SPLIT=1 PROBE_VARIANTS=w2,w3,w4 timeout 300 python tools/tc_probe.py c2 2>&1 | grep shape
