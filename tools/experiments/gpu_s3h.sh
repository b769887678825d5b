# K1 single-pass packer (pack_fused_kernel, 16-segment tiles, one quad per loop trip) vs scan + scatter (pack2k build): parity + times
# (see gpu_s3i.sh for the same A/B after unrolling the scatter loop)
