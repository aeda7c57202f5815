# round 2: GPU suite with the out-of-line checker
O=gpurun_out/r02ab
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
LBM_LIBRARY=paper_1007_1388_b200/liblbm_b200_checked.so timeout 900 python tools/sanitize_cases.py > $O/checked_cases.log 2>&1; echo "rc=$?" >> $O/checked_cases.log
LBM_CHECKED_INJECT=1 LBM_LIBRARY=paper_1007_1388_b200/liblbm_b200_checked.so timeout 300 python tools/sanitize_cases.py --first > $O/checked_inject.log 2>&1; echo "rc=$?" >> $O/checked_inject.log
echo done
