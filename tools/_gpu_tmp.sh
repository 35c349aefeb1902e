echo "== REC12 (main)"; timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py -m gpu -q -x -p no:cacheprovider -k "config2_settings" -s 2>&1 | grep "48^2\|passed\|failed"
echo "== G/H"; PMGB_LIB=$PWD/paper_2202_09733_b200/libpmgflow_b200_gh.so timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py -m gpu -q -x -p no:cacheprovider -k "config2_settings" -s 2>&1 | grep "48^2\|passed\|failed"
echo "== rect tests (main)"; timeout 900 python -m pytest tests/test_gpu_rect_path.py -m gpu -q -p no:cacheprovider 2>&1 | tail -8
