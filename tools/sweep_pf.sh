for PF in ${PFLIST:-none 0,s}; do
  if [ $PF = none ]; then unset PERSEUS_PREFETCH; else export PERSEUS_PREFETCH=$PF; fi
  echo "PF=$PF"; SLIST="4096 8192" bash tools/diag1.sh
done
