# A/B of two variant libraries on a plan, then GPU tests (-k) on the second (dev tool)
# usage: bash tools/ab_var.sh A B "plan" "pytest -k expr"
A=$1; B=$2; PLAN=$3; K=$4
rm -f gpurun_out/ab.log gpurun_out/abtest.log
for v in $A $B $A $B; do WK_LIB_PATH=variants/libwk_$v.so WK_AB_TAG=$v timeout 300 python tools/ab_time.py $PLAN >> gpurun_out/ab.log 2>&1; done
WK_LIB_PATH=variants/libwk_$B.so timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/abtest.log 2>&1
