// Probe: cuFile (GPUDirect Storage) on the GPU box — driver open, mode (native or
// compatibility), and the throughput of reading a 640 MiB file straight into HBM
// (cuFileRead) vs a parallel buffered pread into pinned host memory + one H2D copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/gds_probe scripts/micro/gds_probe.cu -lcufile
//   /tmp/gds_probe /tmp/gds_probe.bin
#include <cufile.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static void drop(const char* p) {
  int fd = open(p, O_RDONLY);
  fdatasync(fd);
  posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);
  close(fd);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const char* path = argc > 1 ? argv[1] : "/tmp/gds_probe.bin";
  const size_t n = 640ull << 20;
  {  // the file
    std::vector<char> buf(64 << 20, 7);
    int fd = open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
    for (size_t o = 0; o < n; o += buf.size()) (void)!write(fd, buf.data(), buf.size());
    fsync(fd);
    close(fd);
  }
  void* dev = nullptr;
  cudaMalloc(&dev, n);
  printf("{\"file_written\": 1, ");
  CUfileError_t st = cuFileDriverOpen();
  printf("\"driver_open\": %d", st.err);
  CUfileDrvProps_t props;
  memset(&props, 0, sizeof(props));
  if (st.err == CU_FILE_SUCCESS && cuFileDriverGetProperties(&props).err == CU_FILE_SUCCESS)
    printf(", \"nvfs_major\": %u, \"nvfs_minor\": %u, \"dstatus_flags\": %u, \"dcontrol_flags\": %u",
           props.nvfs.major_version, props.nvfs.minor_version, props.nvfs.dstatusflags, props.nvfs.dcontrolflags);
  for (int direct = 1; direct >= 0; --direct) {
    drop(path);
    int fd = open(path, O_RDONLY | (direct ? O_DIRECT : 0));
    if (fd < 0) {
      printf(", \"open_%s\": \"failed\"", direct ? "direct" : "buffered");
      continue;
    }
    CUfileDescr_t d;
    memset(&d, 0, sizeof(d));
    d.handle.fd = fd;
    d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
    CUfileHandle_t h;
    CUfileError_t r = cuFileHandleRegister(&h, &d);
    printf(", \"register_%s\": %d", direct ? "direct" : "buffered", r.err);
    if (r.err == CU_FILE_SUCCESS) {
      cuFileBufRegister(dev, n, 0);
      const double t0 = now();
      // 8 threads of 80 MiB each, like the host read path
      std::vector<std::thread> th;
      std::vector<ssize_t> got(8);
      for (int i = 0; i < 8; ++i)
        th.emplace_back([&, i] { got[i] = cuFileRead(h, dev, n / 8, (off_t)(i * (n / 8)), (off_t)(i * (n / 8))); });
      for (auto& t : th) t.join();
      cudaDeviceSynchronize();
      const double dt = now() - t0;
      ssize_t tot = 0;
      for (auto g : got) tot += g > 0 ? g : 0;
      printf(", \"cufile_%s_GBps\": %.2f, \"cufile_%s_bytes\": %zd", direct ? "direct" : "buffered", n / dt / 1e9,
             direct ? "direct" : "buffered", tot);
      cuFileBufDeregister(dev);
      cuFileHandleDeregister(h);
    }
    close(fd);
  }
  {  // baseline: parallel buffered pread into pinned memory, then one H2D
    void* host = nullptr;
    cudaHostAlloc(&host, n, cudaHostAllocDefault);
    drop(path);
    const double t0 = now();
    int fd = open(path, O_RDONLY);
    std::vector<std::thread> th;
    for (int i = 0; i < 8; ++i)
      th.emplace_back([&, i] {
        size_t off = i * (n / 8), end = off + n / 8;
        while (off < end) {
          ssize_t k = pread(fd, static_cast<char*>(host) + off, end - off, off);
          if (k <= 0) break;
          off += k;
        }
      });
    for (auto& t : th) t.join();
    close(fd);
    const double t1 = now();
    cudaMemcpy(dev, host, n, cudaMemcpyHostToDevice);
    const double t2 = now();
    printf(", \"pread8_GBps\": %.2f, \"h2d_GBps\": %.2f, \"pread_plus_h2d_GBps\": %.2f", n / (t1 - t0) / 1e9,
           n / (t2 - t1) / 1e9, n / (t2 - t0) / 1e9);
    cudaFreeHost(host);
  }
  printf("}\n");
  cuFileDriverClose();
  unlink(path);
  return 0;
}
