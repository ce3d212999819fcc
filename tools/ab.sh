# A/B of an env switch on the same box: A=unset, B=$ABVAR=$ABVAL, alternated
for r in 1 2; do
  for v in "" "$ABVAL"; do
    if [ -z "$v" ]; then unset $ABVAR; else export $ABVAR=$v; fi
    echo "$ABVAR=$v"; SLIST="${SLIST:-4096 8192}" bash tools/diag1.sh
  done
done
