// tcp.cpp -- see tcp.hpp.
#include "tcp.hpp"

#include <arpa/inet.h>
#include <fcntl.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cerrno>
#include <cstdlib>
#include <cstring>

namespace gpcx::tcp {

namespace {

[[noreturn]] void sys_fail(Errc code, const std::string& what) {
  fail(code, what + ": " + std::strerror(errno));
}

void make_nonblocking(int fd) {
  const int fl = ::fcntl(fd, F_GETFL, 0);
  if (fl < 0 || ::fcntl(fd, F_SETFL, fl | O_NONBLOCK) < 0) sys_fail(Errc::IoError, "fcntl");
}

// Per-connection options: no Nagle delay on the 260-byte frames.  Socket
// buffers stay under the kernel's autotuning -- fixed 8 MiB SO_SNDBUF /
// SO_RCVBUF measured 61-63 vs 66-68 chains/s on C5's 64 loopback
// connections (profiles/r1/tcp_buffers_ab.txt); GPCX_TCP_BUF=<bytes> pins
// them for A/B runs.
void set_conn_options(int fd) {
  const int on = 1;
  ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &on, sizeof(on));
  static const int pinned_buf = [] {
    const char* v = std::getenv("GPCX_TCP_BUF");
    return v != nullptr ? std::atoi(v) : 0;
  }();
  if (pinned_buf > 0) {
    ::setsockopt(fd, SOL_SOCKET, SO_SNDBUF, &pinned_buf, sizeof(pinned_buf));
    ::setsockopt(fd, SOL_SOCKET, SO_RCVBUF, &pinned_buf, sizeof(pinned_buf));
  }
}

}  // namespace

void Fd::reset(int fd) {
  if (fd_ >= 0) ::close(fd_);
  fd_ = fd;
}

std::string peer_name(int fd) {
  sockaddr_in sa{};
  socklen_t len = sizeof(sa);
  if (::getpeername(fd, reinterpret_cast<sockaddr*>(&sa), &len) != 0) return "?";
  char text[INET_ADDRSTRLEN] = {};
  if (::inet_ntop(AF_INET, &sa.sin_addr, text, sizeof(text)) == nullptr) return "?";
  return std::string(text) + ":" + std::to_string(ntohs(sa.sin_port));
}

Conn::Conn(Fd fd, std::chrono::milliseconds read_idle, std::chrono::milliseconds write_idle)
    : fd_(std::move(fd)), read_idle_(read_idle), write_idle_(write_idle) {
  peer_ = peer_name(fd_.get());
}

void Conn::wait(short events) {
  pollfd p{fd_.get(), events, 0};
  const auto idle = events == POLLIN ? read_idle_ : write_idle_;
  const int budget = idle.count() < 0 ? -1 : static_cast<int>(idle.count());
  for (;;) {
    const int r = ::poll(&p, 1, budget);
    if (r > 0) return;  // ready, or an error / hangup the next syscall reports
    if (r == 0) fail(Errc::TimedOut, events == POLLIN ? "read timed out" : "write timed out");
    if (errno != EINTR) sys_fail(Errc::IoError, "poll");
  }
}

long Conn::try_read(std::span<std::uint8_t> out) {
  for (;;) {
    const ssize_t n = ::recv(fd_.get(), out.data(), out.size(), 0);
    if (n >= 0) return static_cast<long>(n);
    if (errno == EINTR) continue;
    if (errno == EAGAIN || errno == EWOULDBLOCK) return -1;
    sys_fail(Errc::IoError, "recv");
  }
}

std::size_t Conn::read_some(std::span<std::uint8_t> out) {
  if (out.empty()) return 0;
  for (;;) {
    const long n = try_read(out);
    if (n >= 0) return static_cast<std::size_t>(n);
    wait(POLLIN);
  }
}

void Conn::write_all(std::span<const std::uint8_t> data) {
  while (!data.empty()) {
    const ssize_t n = ::send(fd_.get(), data.data(), data.size(), MSG_NOSIGNAL);
    if (n > 0) {
      data = data.subspan(static_cast<std::size_t>(n));
      continue;
    }
    if (n < 0 && errno == EINTR) continue;
    if (n < 0 && (errno == EAGAIN || errno == EWOULDBLOCK)) {
      wait(POLLOUT);
      continue;
    }
    sys_fail(Errc::IoError, "send");
  }
}

Conn dial(const std::string& host, std::uint16_t port) {
  addrinfo want{};
  want.ai_family = AF_INET;
  want.ai_socktype = SOCK_STREAM;
  addrinfo* found = nullptr;
  const std::string where = host + ":" + std::to_string(port);
  if (const int rc = ::getaddrinfo(host.c_str(), std::to_string(port).c_str(), &want, &found))
    fail(Errc::ConnectFailed, where + ": " + gai_strerror(rc));
  std::string last = "no address";
  Fd fd;
  for (const addrinfo* a = found; a != nullptr; a = a->ai_next) {
    Fd s(::socket(a->ai_family, a->ai_socktype | SOCK_CLOEXEC, a->ai_protocol));
    if (!s) {
      last = std::strerror(errno);
      continue;
    }
    int rc;
    do rc = ::connect(s.get(), a->ai_addr, a->ai_addrlen);
    while (rc != 0 && errno == EINTR);
    if (rc == 0) {
      fd = std::move(s);
      break;
    }
    last = std::strerror(errno);
  }
  ::freeaddrinfo(found);
  if (!fd) fail(Errc::ConnectFailed, where + ": " + last);
  set_conn_options(fd.get());
  make_nonblocking(fd.get());
  return Conn(std::move(fd));
}

Listener::Listener(const std::string& bind_addr, std::uint16_t port) {
  sockaddr_in sa{};
  sa.sin_family = AF_INET;
  sa.sin_port = htons(port);
  const std::string where = bind_addr + ":" + std::to_string(port);
  if (::inet_pton(AF_INET, bind_addr.c_str(), &sa.sin_addr) != 1)
    fail(Errc::BindFailed, "bad bind address " + bind_addr);
  fd_.reset(::socket(AF_INET, SOCK_STREAM | SOCK_NONBLOCK | SOCK_CLOEXEC, 0));
  if (!fd_) sys_fail(Errc::BindFailed, "socket");
  const int on = 1;
  ::setsockopt(fd_.get(), SOL_SOCKET, SO_REUSEADDR, &on, sizeof(on));
  if (::bind(fd_.get(), reinterpret_cast<const sockaddr*>(&sa), sizeof(sa)) != 0)
    sys_fail(Errc::BindFailed, where);
  if (::listen(fd_.get(), SOMAXCONN) != 0) sys_fail(Errc::BindFailed, where);
  socklen_t len = sizeof(sa);
  port_ = ::getsockname(fd_.get(), reinterpret_cast<sockaddr*>(&sa), &len) == 0
              ? ntohs(sa.sin_port)
              : port;
}

Fd Listener::accept_one() {
  for (;;) {
    const int c = ::accept4(fd_.get(), nullptr, nullptr, SOCK_NONBLOCK | SOCK_CLOEXEC);
    if (c >= 0) {
      set_conn_options(c);
      return Fd(c);
    }
    if (errno == EINTR || errno == ECONNABORTED) continue;
    return Fd();  // EAGAIN (queue drained) or a transient error (EMFILE, ENOBUFS)
  }
}

}  // namespace gpcx::tcp
