# IMGS reducer / pipe variants, alternated on one box (per MGS step vs k, config-2 recipe)
for rep in 1 2; do
for v in "X=1" "RBG_IMGS_PRE=0" "RBG_IMGS_CTAS=8" "RBG_IMGS_BULK=1"; do
  echo "== $v (rep $rep)"; env $v python scripts/imgs_scaling.py 40960 300 2>&1 | tail -3
done
done
