L=$PWD/tools/variants/exp/libbmc_b200.so
for kb in 1 2 3 4 6 8; do echo "kblk=$kb"; BMC_KBLK=$kb VARIANT=k$kb VARIANT_LIB=$L timeout 300 python tools/time_me.py c2 8 2>&1 | tail -1; done
echo nosea; BMC_NO_SEA=1 VARIANT=nosea VARIANT_LIB=$L timeout 300 python tools/time_me.py c2 8 2>&1 | tail -1
for pm in 1 2 4; do echo "persist=$pm"; BMC_PERSIST=$pm VARIANT=p$pm VARIANT_LIB=$L timeout 300 python tools/time_me.py c2 8 2>&1 | tail -1; done
for pm in 1 2; do echo "persist=$pm kblk4"; BMC_KBLK=4 BMC_PERSIST=$pm VARIANT=p$pm VARIANT_LIB=$L timeout 300 python tools/time_me.py c2 8 2>&1 | tail -1; done
