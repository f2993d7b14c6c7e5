# A/B of kernel selections on one library (dev tool)
# usage: bash tools/ab_env.sh "ENV1=a ENV2=b|ENV1=c" "plan" [lib]
IFS='|' read -ra VARS <<< "$1"; PLAN=$2
for rep in 1 2; do for v in "${VARS[@]}"; do env $v WK_AB_TAG="$v" timeout 600 python tools/ab_time.py $PLAN >> gpurun_out/ab.log 2>&1; done; done
