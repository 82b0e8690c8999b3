// Two processes on one GPU: the child spins in a kernel on a flag that lives in
// the parent's memory (CUDA IPC); the parent sets it from a kernel a second
// later. Checks that cross-process spin waits make progress (time-slicing) and
// see the release store. Build: nvcc -gencode arch=compute_100a,code=sm_100a ipc_spin.cu -o ipc_spin
#include <cstdio>
#include <cuda_runtime.h>
#include <sys/wait.h>
#include <unistd.h>

__global__ void spin(int* f, int want, long long* cycles) {
  long long t0 = clock64();
  int v;
  do {
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  } while (v < want);
  *cycles = clock64() - t0;
}
__global__ void set(int* f, int v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

int main() {
  int fd[2];
  if (pipe(fd)) return 1;
  pid_t pid = fork();
  if (pid == 0) {  // child
    cudaIpcMemHandle_t h;
    if (read(fd[0], &h, sizeof h) != sizeof h) return 2;
    int* f = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle((void**)&f, h, cudaIpcMemLazyEnablePeerAccess);
    long long* c;
    cudaMalloc(&c, 8);
    spin<<<1, 1>>>(f, 1, c);
    e = cudaDeviceSynchronize();
    long long hc = 0;
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    std::printf("child: spin done (%s), %lld cycles\n", cudaGetErrorString(e), hc);
    return 0;
  }
  int* f;
  cudaMalloc(&f, 4);
  cudaMemset(f, 0, 4);
  cudaIpcMemHandle_t h;
  cudaIpcGetMemHandle(&h, f);
  if (write(fd[1], &h, sizeof h) != sizeof h) return 3;
  sleep(2);
  set<<<1, 1>>>(f, 1);
  cudaDeviceSynchronize();
  std::printf("parent: flag set\n");
  int st = 0;
  waitpid(pid, &st, 0);
  std::printf("parent: child exited %d\n", st);
  return 0;
}
