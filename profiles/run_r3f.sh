for v in head new head new; do TGP_LIB=profiles/ablib/libtgp_$v.so timeout 60 python profiles/step_breakdown.py 2>&1 | head -1 | sed "s/^/$v /"; done
timeout 100 python -m pytest tests/test_gpu_parity.py -x -q --timeout 60 -k "two_steps or c2_small" 2>&1 | tail -1
