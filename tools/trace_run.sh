mkdir -p gpurun_out
for cta in 19 0 1; do
PSLR_LIB=$PWD/lib_variants/trace3/libpslr.so PSLR_TRACE=1 PSLR_TRACE_CTA=$cta timeout 300 python tools/trace_apply.py cfg5 > gpurun_out/trace3_cta$cta.log 2>&1
done
echo done
