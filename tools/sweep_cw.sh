for CW in ${CWLIST:-1 2 4 6}; do
  export PERSEUS_COMBINE_WARPS=$CW
  echo "CW=$CW"; SLIST="4096" bash tools/diag1.sh
done
bash tools/tl.sh
