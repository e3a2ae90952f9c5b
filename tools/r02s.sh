for wl in crbd seir fig3; do bash tools/variants.sh $wl "" "-DSMC_DIAG_FUSED_NO_GATHER=1"; done
