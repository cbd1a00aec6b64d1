for v in "X=1" "RBG_IMGS_PRE=0" "RBG_IMGS_CTAS=8" "RBG_IMGS_CTAS=8 RBG_IMGS_PRE=0"; do
  echo "== $v"; env $v python scripts/imgs_scaling.py 40960 300 2>&1 | tail -4
done
