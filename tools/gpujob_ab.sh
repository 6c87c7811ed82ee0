# developer A/B: base library vs the variants named in $@ (C2 device time per application)
bash tools/variants_run.sh "$@"
bash tools/variants_run.sh "$@"
