for wl in seir fig3 stackf; do
  bash tools/variants.sh $wl "" "-DSMC_PROP_THREADS=128" "-DSMC_PROP_THREADS=64" "-DSMC_PROP_THREADS=32"
done
