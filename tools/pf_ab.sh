# L2 bulk prefetch A/B over the configs (dev tool): default rule, forced off, forced on
rm -f gpurun_out/pf_ab.log
PLAN="c2:lsrk45:50 c2:ader_hdg:50 c3:ader_hdg:10 c4:ader_hdg:5 c4:lsrk45:5 c5:ader_hdg:5"
for pf in auto 0 1; do
  if [ $pf = auto ]; then E=; else E="WK_L2PF=$pf"; fi
  env $E WK_AB_TAG=pf$pf timeout 600 python tools/ab_time.py $PLAN >> gpurun_out/pf_ab.log 2>&1
done
