"""Cold sequential-read throughput of the box's scratch disk: buffered parallel pread
(page cache dropped) vs O_DIRECT parallel pread, 1 GiB file, 1/4/8 threads."""
import json, os, tempfile, threading, time, mmap

n = 1 << 30
d = tempfile.mkdtemp(prefix="rdkv_disk_")
path = os.path.join(d, "f.bin")
with open(path, "wb") as f:
    blk = os.urandom(1 << 24)
    for _ in range(n // len(blk)):
        f.write(blk)
    f.flush(); os.fsync(f.fileno())
out = {"dir": d}


def drop():
    fd = os.open(path, os.O_RDONLY)
    os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    os.close(fd)


def run(threads, direct):
    drop()
    flags = os.O_RDONLY | (os.O_DIRECT if direct else 0)
    fd = os.open(path, flags)
    chunk = n // threads
    def work(i):
        buf = mmap.mmap(-1, 1 << 22)  # page-aligned 4 MiB buffer
        off, end = i * chunk, (i + 1) * chunk
        while off < end:
            k = os.preadv(fd, [buf], off)
            if k <= 0:
                break
            off += k
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts: t.start()
    for t in ts: t.join()
    dt = time.perf_counter() - t0
    os.close(fd)
    return n / dt / 1e9

for th in (1, 4, 8):
    out[f"buffered_{th}t_GBps"] = run(th, False)
    out[f"direct_{th}t_GBps"] = run(th, True)
os.remove(path)
print(json.dumps(out))
