for d in 798 1310 30; do echo "dbg=$d"; TMG_FFP=4 TMG_FFP4_DBG=$d timeout 120 python tools/ffp_probe.py config5-L4 1 2>&1 | tail -1; done
