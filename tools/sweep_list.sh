for c in c2 c3 c1; do
  run $c default ""
done
