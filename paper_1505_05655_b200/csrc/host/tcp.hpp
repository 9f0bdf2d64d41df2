// tcp.hpp -- the executor's TCP transport.
//
// Every socket is non-blocking from the moment it exists.  The front end's
// reactor (server.cpp) multiplexes connections that are still sending their
// 260-byte header over one epoll set; once a request is admitted, the stage
// that owns the connection does its payload / response I/O through Conn,
// whose reads and writes wait with poll() against a per-operation idle
// budget.  The wire contract is the reference's (proj/include/gpc/net.hpp:
// 16-62): an idle peer surfaces as TimedOut, an orderly close before the
// expected bytes as a zero read (-> Truncated in wire::read_exact).  Unlike
// the reference, writes are bounded too, by their own longer stall budget
// (the server uses max(idle, 60 s)): a client that stops reading its
// response cannot pin a send thread forever, while one that merely pauses
// is not cut off at the read idle timeout.  The listen backlog is
// SOMAXCONN, not 64 (proj/src/net.cpp:128).
#pragma once

#include <chrono>
#include <cstdint>
#include <span>
#include <string>

#include "wire.hpp"

namespace gpcx::tcp {

// Owning file descriptor.
class Fd {
 public:
  Fd() = default;
  explicit Fd(int fd) : fd_(fd) {}
  ~Fd() { reset(); }
  Fd(Fd&& o) noexcept : fd_(o.release()) {}
  Fd& operator=(Fd&& o) noexcept {
    if (this != &o) reset(o.release());
    return *this;
  }
  Fd(const Fd&) = delete;
  Fd& operator=(const Fd&) = delete;
  int get() const { return fd_; }
  int release() {
    const int f = fd_;
    fd_ = -1;
    return f;
  }
  void reset(int fd = -1);
  explicit operator bool() const { return fd_ >= 0; }

 private:
  int fd_ = -1;
};

// One connected stream socket (non-blocking underneath).  `read_idle` /
// `write_idle` bound how long a single read / write may wait for the peer;
// negative = forever.
class Conn : public wire::ByteStream {
 public:
  Conn() = default;
  explicit Conn(Fd fd, std::chrono::milliseconds read_idle = std::chrono::milliseconds(-1),
                std::chrono::milliseconds write_idle = std::chrono::milliseconds(-1));
  std::size_t read_some(std::span<std::uint8_t> out) override;  // 0 = peer closed
  void write_all(std::span<const std::uint8_t> data) override;
  // Non-blocking read attempt: bytes read, 0 on orderly close, -1 when
  // nothing is available yet.  Errors throw IoError.
  long try_read(std::span<std::uint8_t> out);

  int fd() const { return fd_.get(); }
  const std::string& peer() const { return peer_; }
  void close() { fd_.reset(); }

 private:
  void wait(short events);  // TimedOut after the direction's budget
  Fd fd_;
  std::string peer_;
  std::chrono::milliseconds read_idle_{-1}, write_idle_{-1};
};

// Blocking-semantics client connect (ConnectFailed); `host` is a name or
// dotted quad, IPv4.
Conn dial(const std::string& host, std::uint16_t port);

// Non-blocking listening socket (BindFailed).  port 0 = ephemeral.
class Listener {
 public:
  Listener(const std::string& bind_addr, std::uint16_t port);
  int fd() const { return fd_.get(); }
  std::uint16_t port() const { return port_; }
  // Next pending connection, or an empty Fd when none is queued.
  Fd accept_one();

 private:
  Fd fd_;
  std::uint16_t port_ = 0;
};

std::string peer_name(int fd);

}  // namespace gpcx::tcp
