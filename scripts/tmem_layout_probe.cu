// Which (TMEM lane, column) each thread's registers hold for tcgen05.ld 16x256b / 16x128b /
// 16x64b: warp 0 writes value = 1000 * lane + column with the 32x32b shape (thread t <->
// lane t), then reads it back with the 16-lane shapes (lane base 0).
#include <cstdint>
#include <cstdio>

__global__ void probe(int* out) {
  __shared__ uint32_t tbase_s;
  const int t = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n"
               :: "r"((uint32_t)__cvta_generic_to_shared(&tbase_s)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase_s;
  uint32_t v[8];
  for (int h = 0; h < 2; ++h) {
    for (int c = 0; c < 8; ++c) v[c] = 1000 * t + 8 * h + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                 :: "r"(tb + 8 * h), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  uint32_t x2[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(x2[0]), "=r"(x2[1]), "=r"(x2[2]), "=r"(x2[3]), "=r"(x2[4]), "=r"(x2[5]), "=r"(x2[6]), "=r"(x2[7]) : "r"(tb));
  uint32_t a[4], b[2], c1;
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(tb));
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];\n" : "=r"(b[0]), "=r"(b[1]) : "r"(tb));
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];\n" : "=r"(c1) : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  for (int i = 0; i < 4; ++i) out[t * 8 + i] = a[i];
  out[t * 8 + 4] = b[0];
  out[t * 8 + 5] = b[1];
  out[t * 8 + 6] = c1;
  for (int i = 0; i < 8; ++i) out[256 + t * 8 + i] = x2[i];
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" :: "r"(tb));
}

int main() {
  int* d;
  cudaMalloc(&d, 2 * 32 * 8 * 4);
  probe<<<1, 32>>>(d);
  int h[2 * 32 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %d\n", (int)cudaGetLastError());
  printf("thread: 16x256b regs (lane*1000+col) | 16x128b | 16x64b\n");
  for (int t = 0; t < 32; ++t)
    printf("%2d: %5d %5d %5d %5d | %5d %5d | %5d\n", t, h[t * 8], h[t * 8 + 1], h[t * 8 + 2],
           h[t * 8 + 3], h[t * 8 + 4], h[t * 8 + 5], h[t * 8 + 6]);
  printf("16x256b.x2 regs:\n");
  for (int t = 0; t < 8; ++t) {
    printf("%2d:", t);
    for (int i = 0; i < 8; ++i) printf(" %5d", h[256 + t * 8 + i]);
    printf("\n");
  }
  return 0;
}
