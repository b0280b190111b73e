"""Make a stamped copy of attn_prefill.cu (CTA 0, first softmax warp of tile a, lane 0):
per S block: 0 before the S wait, 1 S ready, 2 TMEM loaded, 3 before the P store, 4 P published."""
import sys
src = open(sys.argv[1]).read()
src = src.replace("namespace slx {\nnamespace {\n", "namespace slx {\n__device__ unsigned long long g_dbg[8192];\nnamespace {\n", 1)
T = "blockIdx.x == 0 && threadIdx.x == 96"
src = src.replace("        tc::mbar_wait(s_full(t, sb), (si >> 1) & 1);",
                  f"        if ({T} && si < 1000) g_dbg[si * 8 + 0] = clock64();\n        tc::mbar_wait(s_full(t, sb), (si >> 1) & 1);\n        if ({T} && si < 1000) g_dbg[si * 8 + 1] = clock64();")
src = src.replace("        tmem_ld32(tbase + lane_off + sb * FT_BK + 32, s + 32);",
                  f"        tmem_ld32(tbase + lane_off + sb * FT_BK + 32, s + 32);\n        if ({T} && si < 1000) g_dbg[si * 8 + 2] = clock64() + (s[0] == 1.2345f);")
src = src.replace("        if (pi >= FT_PBUF)   // the P.V that last read this buffer has completed",
                  f"        if ({T} && si < 1001) g_dbg[(si - 1) * 8 + 3] = clock64();\n        if (pi >= FT_PBUF)   // the P.V that last read this buffer has completed")
src = src.replace("        if (lane == 0) tc::mbar_arrive(p_full(t, pb));",
                  f"        if ({T} && si < 1001) g_dbg[(si - 1) * 8 + 4] = clock64();\n        if (lane == 0) tc::mbar_arrive(p_full(t, pb));")
src = src.replace("          ++tw;\n        }", "          ++tw;\n        }\n        if (" + T + " && si < 1001) g_dbg[(si - 1) * 8 + 5] = clock64();")
src += '\nextern "C" SLX_API int slx_dbg_copy(void* host, size_t n) {\n  return cudaMemcpyFromSymbol(host, slx::g_dbg, n) == cudaSuccess ? 0 : -5;\n}\n'
open(sys.argv[2], "w").write(src)
