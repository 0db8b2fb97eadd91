timeout 200 python -m pytest tests/test_gpu_stream.py -x -q --timeout 100 2>&1 | tail -2
for v in head new head new; do TGP_LIB=profiles/ablib/libtgp_$v.so timeout 60 python profiles/step_breakdown.py 2>&1 | head -4 | sed "s/^/$v /"; done
