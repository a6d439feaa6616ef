for n in 1 2 3 4 8; do echo "per_sm=$n"; BMC_CHAIN_PER_SM=$n VARIANT_LIB=$PWD/tools/variants/exp/libbmc_b200.so timeout 120 python tools/step_probe.py c2gop; done
python tools/step_probe.py c2gop
