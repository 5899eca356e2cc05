/*
 * pinn_dd.h -- C ABI of the B200-native per-subdomain training step of parallel
 * cPINN / XPINN (Shukla, Jagtap & Karniadakis, arXiv 2104.10013).
 *
 * Citation key: P:n = PAPER.md line n (LaTeX source of the paper).
 *
 * One handle owns the subdomains Omega_q placed on ONE GPU (one process per
 * GPU).  For every owned subdomain it holds the network parameters Theta_q =
 * {W^k, b^k, a^k}, the Adam state and borrowed pointers to
 * the subdomain's point sets {x_F}, {x_u}, {x_I}.  The calls follow the
 * red / green / optimisation stages of Algorithm 1:
 *
 *   pinn_dd_interface_payload  red, lines 238-243: u(x_I) and f(x_I).n (cPINN)
 *                              or F(x_I) (XPINN) into the payload buffer
 *   (exchange)                 green, lines 244-265: the caller moves payload
 *                              rows of cut edges between ranks (torch.distributed
 *                              / NCCL); intra-GPU neighbours need nothing
 *   pinn_dd_loss_grad          line 253/261: J(Theta_q) of Eq. (5)/(6) and
 *                              dJ/dTheta_q with neighbour values held constant
 *   pinn_dd_adam               lines 266-267: one Adam step per subdomain
 *   pinn_dd_step               all of the above for handles without remote
 *                              neighbours, n_iters times, CUDA-graph replayed
 *   pinn_dd_predict            Eq. (4) stitched solution
 *
 * Conventions
 * -----------
 * - All bulk arrays are DEVICE pointers, float32, caller-owned and BORROWED:
 *   they must stay valid and unchanged until pinn_dd_destroy.  Host arrays in
 *   the descriptor are deep-copied by pinn_dd_create.
 * - Coordinates: x1 = x and x2 = t (Burgers, "time as one component of x")
 *   or x2 = y (Poisson / heat / NS).  Arrays are SoA: coords[2][n_points].
 * - Point order inside the handle: subdomain by subdomain; inside subdomain q
 *   (points [sub_point_offset[q], sub_point_offset[q+1])): first the N_F
 *   residual points, then the N_u training points, then the interface points
 *   edge segment by edge segment (segments [sub_seg_offset[q],
 *   sub_seg_offset[q+1]) of the seg_* arrays, seg_n[s] points each).
 * - Parameters use the layer-major packing W^1, b^1, a^1, ..., W^{L-1},
 *   b^{L-1}, a^{L-1}, W^L, b^L with W^k row-major N_k x N_{k-1} (the layout of
 *   pinn_dd_n_params); internally the library pads each tensor to 16 bytes.
 * - Every call returns a status and never throws or aborts across the ABI;
 *   pinn_dd_last_error returns the message of the last failing call.
 *   Asynchronous CUDA errors surface at the next call that synchronises.
 * - Calls are stream-ordered on desc->stream.  Only calls with a HOST output
 *   (pinn_dd_step with loss_host != NULL, pinn_dd_get_step) synchronise.
 */
#ifndef PINN_DD_H
#define PINN_DD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pinn_dd pinn_dd; /* opaque, one per process (GPU) */

typedef enum {
  PINN_DD_OK = 0,
  PINN_DD_EINVAL = 1,        /* shape / count / pointer mismatch, cPINN with a time-axis interface */
  PINN_DD_EUNSUPPORTED = 2,  /* (width, n_hidden, d_out, activation) not compiled in */
  PINN_DD_ECUDA = 3,         /* CUDA runtime error; message carries cudaGetErrorString */
  PINN_DD_ENCCL = 4,         /* NCCL unavailable or an NCCL call failed (message carries NCCL's text) */
  PINN_DD_ENONFINITE = 5,    /* a loss J_q or gradient is NaN/Inf (message names the subdomain) */
  PINN_DD_EPROTOCOL = 6      /* malformed twin / exchange plan; remote twins without a transport */
} pinn_dd_status;

/* HYBRID ("cPINN in space + XPINN in time"): per interface edge, normal-flux
   continuity on x1-normal edges (cPINN, Eq. 5) and residual continuity on
   x2-normal edges (XPINN, Eq. 6). */
enum { PINN_DD_METHOD_PINN = 0, PINN_DD_METHOD_CPINN = 1, PINN_DD_METHOD_XPINN = 2, PINN_DD_METHOD_HYBRID = 3 };
/* P:313-316 Burgers; P:823-829 heat (K known; POISSON = K==1 with u* = sin(pi x) sin(pi y));
   P:415-417 steady incompressible NS (outputs u, v, p); P:821-871 inverse heat conduction
   HEAT_INV: one net per region with outputs (T, K), F = div(K grad T) - f, f = 4 exp(-0.1 y). */
enum { PINN_DD_PDE_BURGERS = 0, PINN_DD_PDE_POISSON = 1, PINN_DD_PDE_HEAT = 2, PINN_DD_PDE_NS = 3,
       PINN_DD_PDE_HEAT_INV = 4 };
enum { PINN_DD_ACT_TANH = 0, PINN_DD_ACT_SIN = 1, PINN_DD_ACT_COS = 2 };
/* Eq. (4) geometry of the decomposition: which subdomains own a point. */
enum { PINN_DD_GEOM_NONE = 0,     /* no geometry: only pinn_dd_predict_owners            */
       PINN_DD_GEOM_BOXES = 1,    /* Cartesian cells [lo_x, hi_x] x [lo_y, hi_y] (closed)   */
       PINN_DD_GEOM_VORONOI = 2   /* nearest-seed cells clipped by a simple polygon (C5)    */ };
/* pinn_dd_predict modes */
enum { PINN_DD_PREDICT_STITCHED = 0,  /* Eq. (4): average of the owners' nets, weight 1/S       */
       PINN_DD_PREDICT_OWNER = 1 };   /* the net of the lowest-id owner only (weight 1)         */

/* flags */
#define PINN_DD_FLAG_GRAPH        1  /* pinn_dd_step replays a captured CUDA graph */
#define PINN_DD_FLAG_GLOBAL_STASH 2  /* keep the reverse-mode stash in global memory instead of TMEM (debug) */
#define PINN_DD_FLAG_TIMING       4  /* record per-kernel CUDA events (see pinn_dd_kernel_times) */
#define PINN_DD_FLAG_PEER_STORES 16  /* remote twins move by stores into the neighbours' memory inside
                                        the fused launch (pinn_dd_ipc_export / pinn_dd_connect_peers) */
#define PINN_DD_FLAG_TF32         8  /* width-80 nets: hidden-layer contractions on the tensor cores
                                        (tcgen05.mma kind::tf32, single-pass TF32 products, FP32
                                        accumulation; looser tolerance, DESIGN.md 6 / 11).  Compiled
                                        for [2, 80x5, 3] and [2, 80x3, 2] (per-subdomain activation);
                                        other shapes: PINN_DD_EUNSUPPORTED */

/* Status bits of one loss + gradient evaluation (loss column 5, per subdomain).
   A slope a^k that reaches 0 (set_params, or Adam) makes its gradient NaN. */
#define PINN_DD_STATUS_J_NONFINITE      1
#define PINN_DD_STATUS_GRAD_NONFINITE   2
#define PINN_DD_STATUS_SLOPE_NONFINITE  4
#define PINN_DD_STATUS_SLOPE_ZERO       8

/* Per-subdomain hyper-parameters, P:151-161 (loss weights) and P:286 (Adam). */
typedef struct {
  float w_u;     /* W_u   data-mismatch weight                       */
  float w_f;     /* W_F   residual weight                            */
  float w_i;     /* W_I   average-solution interface weight          */
  float w_if;    /* W_Iflux (cPINN) or W_IF (XPINN) interface weight */
  float lr;      /* Adam learning rate                               */
  float beta1, beta2, eps;
} pinn_dd_hparams;

typedef struct {
  /* ---- problem ---------------------------------- */
  int32_t method;      /* PINN_DD_METHOD_*                                   */
  int32_t pde;         /* PINN_DD_PDE_*                                      */
  int32_t activation;  /* PINN_DD_ACT_* (all subdomains unless sub_activation) */
  int32_t d_in;        /* must be 2                                          */
  int32_t d_out;       /* 1; 3 for NS (u, v, p); 2 for HEAT_INV (T, K)       */
  int32_t width;       /* N_k of every hidden layer                          */
  int32_t n_hidden;    /* L-1 hidden layers                                  */
  float slope_n;       /* n of the adaptive slope n a^k (n = 10)       */
  float nu;            /* Burgers viscosity (0.01/pi)                 */
  float re;            /* NS Reynolds number (100)                    */
  /* ---- subdomains owned by this handle (host arrays, copied) ---------- */
  int32_t n_sub;
  const int32_t* sub_point_offset;  /* [n_sub+1]                              */
  const int32_t* sub_n_res;         /* [n_sub]  N_F                           */
  const int32_t* sub_n_data;        /* [n_sub]  N_u (may be 0)                */
  const int32_t* sub_seg_offset;    /* [n_sub+1] into the seg_* arrays        */
  const pinn_dd_hparams* sub_hparams; /* [n_sub]                              */
  /* ---- interface edge segments (host arrays, copied) ------------------ */
  int32_t n_seg;
  const int32_t* seg_n;      /* [n_seg] N_I of the edge                             */
  const float* seg_normal;   /* [n_seg][2] canonical unit normal of the edge */
  const int64_t* seg_twin;   /* [n_seg] payload slot of the twin (neighbour's copy)
                                of the segment's first point; slots < n_points are
                                local points, slots >= n_points are received rows  */
  /* ---- point table (DEVICE, borrowed) -------------------------------- */
  int64_t n_points;
  int64_t n_recv;            /* payload rows received from other ranks            */
  const float* coords;       /* [2][n_points]                                      */
  const float* target;       /* [d_out][n_points]   training targets u^(i)         */
  const float* mask;         /* [d_out][n_points]   1 = constrained output         */
  const float* init_params;  /* [n_sub][pinn_dd_n_params(...)] packed, or NULL = W = b = 0,
                                a^k = 1/slope_n.  Every a^k must be finite and non-zero
                                (EINVAL): the slope gradient uses a^k dJ/da^k = <W^k, dJ/dW^k> +
                                <b^k, dJ/db^k>, undefined at a^k = 0         */
  /* ---- runtime --------------------------------------------------------- */
  void* stream;              /* cudaStream_t (NULL = legacy default stream)        */
  int32_t flags;             /* PINN_DD_FLAG_*                                     */
  /* ---- data-parallel shards (host, nullable) -------------------------- */
  const int32_t* sub_norm_counts; /* [n_sub][2] (N_F, N_u) used for the 1/N of MSE_F and
                                MSE_u instead of the local counts: a rank holding a shard of
                                a subdomain's points then produces exactly its additive share
                                of J and dJ/dTheta (sum over ranks = the full-data values). */
  /* ---- per-subdomain activation (host, nullable) ---------------------- */
  const int32_t* sub_activation; /* [n_sub] PINN_DD_ACT_* of each subdomain's net (Table 3,
                                P:862-866: tanh / sin / cos per region); NULL = `activation`
                                everywhere.  Mixed values need a network shape compiled with
                                per-subdomain activations (else PINN_DD_EUNSUPPORTED). */
  /* ---- exchange with other ranks (Algorithm 1 green stage; host, copied) ---
     Rows [n_points, n_points + n_recv) of the payload buffer are received from
     other ranks.  With an NCCL transport (nccl_id != NULL) pinn_dd_step runs the
     whole iteration itself -- K2, ncclSend/ncclRecv of the cut-edge rows on an
     internal stream overlapped with K1 over the residual + training points, K1
     over the interface points, K5 -- captured into one CUDA graph.  A peer may be
     this rank itself (loop-back; single-GPU validation of the transport).      */
  int32_t rank;              /* rank of this process in the exchange communicator          */
  int32_t world;             /* communicator size (ignored when nccl_id == NULL)            */
  int32_t n_peers;           /* ranks this handle exchanges rows with                       */
  const int32_t* peer_rank;  /* [n_peers] distinct, ascending                               */
  const int64_t* peer_send_off; /* [n_peers + 1] offsets into send_rows                     */
  const int64_t* send_rows;  /* local interface-point rows (< n_points) sent to each peer, in
                                the order that peer receives them                           */
  const int64_t* peer_recv_row; /* [n_peers] first received row; ranges tile
                                [n_points, n_points + n_recv) in peer order                 */
  const int64_t* peer_recv_n;   /* [n_peers] rows received from each peer                  */
  const void* nccl_id;       /* 128-byte ncclUniqueId (host) shared by the `world` ranks
                                (pinn_dd_nccl_unique_id on one rank, broadcast by the caller);
                                pinn_dd_create then joins the communicator (collective: every
                                rank must call it).  NULL = no transport: the caller moves
                                received rows itself between the phased calls.              */
  /* ---- Eq. (4) geometry (host, copied; optional) -------------------------- */
  int32_t geometry;          /* PINN_DD_GEOM_*                                               */
  int32_t n_geo;             /* subdomains of the WHOLE decomposition described below       */
  const float* geo;          /* BOXES: [n_geo][4] (lo_x, lo_y, hi_x, hi_y); VORONOI: [n_geo][2] seeds */
  const int32_t* geo_local;  /* [n_geo] local subdomain index of each entry, -1 = owned by another rank */
  int32_t n_poly;            /* VORONOI: vertices of the simple domain polygon             */
  const float* poly;         /* [n_poly][2]                                                   */
  float geo_tol;             /* BOXES: a point within geo_tol of a cell is in it (closed cells);
                                VORONOI: seeds whose squared distance is within geo_tol of the
                                nearest one are co-owners (points on interfaces, weight 1/S) */
} pinn_dd_desc;

/* Number of packed parameters of one network [d_in, width x n_hidden, d_out]:
   sum_k (N_k N_{k-1} + N_k) + (L-1) slopes. */
int64_t pinn_dd_n_params(int32_t d_in, int32_t width, int32_t n_hidden, int32_t d_out);

/* Device workspace the handle needs (bytes); the caller allocates it (e.g. a
   torch uint8 tensor) and passes it to pinn_dd_create.  Alignment 256 B. */
pinn_dd_status pinn_dd_workspace_size(const pinn_dd_desc* d, size_t* bytes);

/* Validate the descriptor, plan tiles and chunks, copy the initial parameters
   into the workspace (Adam m = v = 0, t = 0).  The workspace is borrowed. */
pinn_dd_status pinn_dd_create(const pinn_dd_desc* d, void* dev_workspace, size_t ws_bytes,
                              pinn_dd** out);

/* K2: u(x_I) and f(x_I).n (cPINN, Table 1) or F(x_I) (XPINN) of every
   local interface point from the CURRENT parameters into the payload buffer
   (Algorithm 1).  Row r of the buffer holds d_out + n_eq floats. */
pinn_dd_status pinn_dd_interface_payload(pinn_dd* h);

/* Payload buffer [n_points + n_recv][n_fields] (device, library-owned).  Rows
   [0, n_points) are written by pinn_dd_interface_payload; rows [n_points,
   n_points + n_recv) must be filled by the caller's exchange before
   pinn_dd_loss_grad. n_fields = d_out + n_eq (n_eq = 3 for NS, else 1). */
pinn_dd_status pinn_dd_payload_buffer(pinn_dd* h, float** buf, int32_t* n_fields, int64_t* n_rows);

/* K1 + K5(reduce): J(Theta_q) (Eq. 5 cPINN / Eq. 6 XPINN / Eq. 3 if no live
   interface) and g_q = dJ_q/dTheta_q with every neighbour value
   constant, for all local q.  Requires a current payload buffer.
   loss_dev (nullable): device [n_sub][8] = {MSE_u, MSE_F, MSE_uavg,
   MSE_flux|MSE_R, J, status, 0, 0}; status = OR of PINN_DD_STATUS_* bits of
   this evaluation (0 = all finite).  grad_dev (nullable): device [n_sub][n_params]
   packed gradient. */
pinn_dd_status pinn_dd_loss_grad(pinn_dd* h, float* loss_dev, float* grad_dev);

/* The same computation in two stream-ordered halves, so that the payload
   exchange with other ranks overlaps interior compute:
   _interior runs K1 over the residual and training points (it reads no payload
   row and may be enqueued before the exchange completes); _interface runs K1
   over the interface points (needs the complete payload buffer) and K5(reduce)
   with the outputs of pinn_dd_loss_grad.  K1's chunks never mix the two point
   classes, so interior + interface gives pinn_dd_loss_grad's results bit for
   bit. */
pinn_dd_status pinn_dd_loss_grad_interior(pinn_dd* h);
pinn_dd_status pinn_dd_loss_grad_interface(pinn_dd* h, float* loss_dev, float* grad_dev);

/* K5(adam): one bias-corrected Adam step (beta1, beta2, eps, lr per subdomain)
   on every local subdomain with the gradient of the last pinn_dd_loss_grad. */
pinn_dd_status pinn_dd_adam(pinn_dd* h);

/* n_iters x (payload -> [exchange] -> loss+grad -> Adam), one synchronous
   Jacobi iteration each (payloads from the parameters at the start of the
   iteration, Algorithm 1).  Handles with remote twins (n_recv > 0)
   need the NCCL transport (desc nccl_id; else PINN_DD_EPROTOCOL); every rank
   must call pinn_dd_step with the same n_iters.  With PINN_DD_FLAG_GRAPH the
   iteration is captured once into a CUDA graph (exchange included) and
   replayed.  loss_host (nullable):
   host [n_sub][8] breakdown of the LAST iteration (synchronises); a non-zero
   status column (non-finite J or gradient, zero slope) returns
   PINN_DD_ENONFINITE naming the subdomain. */
pinn_dd_status pinn_dd_step(pinn_dd* h, int32_t n_iters, float* loss_host);

/* The library's exchange (NCCL transport only) as a stream-ordered call for the
   phased path: sends the cut-edge rows written by the last
   pinn_dd_interface_payload and receives rows [n_points, n_points + n_recv)
   (ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd on desc->stream).
   Collective over the peers: they must all call it. */
pinn_dd_status pinn_dd_exchange(pinn_dd* h);

/* Peer-store transport (PINN_DD_FLAG_PEER_STORES; Algorithm 1 lines 244-265 fused
   into the step's persistent launch).  Every rank exports its exchange
   region -- per-peer arrival counters (uint64) and payload rows -- as a CUDA IPC
   handle (64 bytes) of the allocation holding it plus byte offsets, the ranks
   trade them (e.g. an all-gather), and each connects to its peers.  Then
   pinn_dd_step runs ONE persistent launch (+ K5) per iteration: payload chunks
   store every cut-edge row straight into the neighbour's receive slot (slot =
   step parity) and release-add the row counts to its arrival counter; the
   interface loss chunks acquire-wait for all peers' rows of the step while the
   interior chunks compute.  Every rank must step in lock-step. */
pinn_dd_status pinn_dd_ipc_export(pinn_dd* h, void* handle64, int64_t* flags_offset, int64_t* rows_offset);
/* For peer i of the exchange plan: handles[i] (64 bytes), the offsets of its
   pinn_dd_ipc_export, peer_row[i] = the peer's first received row from this rank
   (its peer_recv_row), peer_nrecv[i] = the peer's n_recv (slot stride),
   peer_flag[i] = this rank's index among the peer's peers.  A peer whose rank is
   desc->rank is this handle itself (loop-back; its handle is not opened). */
pinn_dd_status pinn_dd_connect_peers(pinn_dd* h, const void* handles, const int64_t* flags_offset,
                                     const int64_t* rows_offset, const int64_t* peer_row,
                                     const int64_t* peer_nrecv, const int32_t* peer_flag);

/* A fresh 128-byte ncclUniqueId (host) for desc->nccl_id (PINN_DD_ENCCL if NCCL
   cannot be loaded). */
pinn_dd_status pinn_dd_nccl_unique_id(void* id128);

/* Stream-ordered copy of the loss breakdown [n_sub][8] (MSE_u, MSE_F,
   MSE_uavg, MSE_if, J_q (Eq. 5/6), status bits, 0, 0) of the last
   loss+grad evaluation into dst (pinned host or device memory, caller-owned).
   No synchronisation and no status check (read the status column, or call
   pinn_dd_step with loss_host); lets a caller pipeline the per-step loss
   read-back with the next step. */
pinn_dd_status pinn_dd_read_loss(pinn_dd* h, float* dst);

/* K6: Eq. (4) stitched solution u(z) = sum_q u_q(z) 1_{Omega_q}(z)
   with the indicator 1 inside Omega_q, 1/S on an interface shared by S
   subdomains and 0 outside every subdomain; the owners of each point are
   classified by the library from desc->geometry (EINVAL without one).  pts:
   device [2][n]; out: device [d_out][n].  mode PINN_DD_PREDICT_STITCHED
   (Eq. 4) or PINN_DD_PREDICT_OWNER (the lowest-id owner's net, weight 1).  S
   counts owners on every rank; a handle adds only its LOCAL owners' terms, so
   with several ranks the caller sums `out` over ranks (e.g. an all-reduce). */
pinn_dd_status pinn_dd_predict(pinn_dd* h, const float* pts, int64_t n, float* out, int32_t mode);

/* Same as pinn_dd_predict(STITCHED) with the caller's classification: owners
   device [n][4] local subdomain ids (-1 = unused), weight 1/(number of ids). */
pinn_dd_status pinn_dd_predict_owners(pinn_dd* h, const float* pts, const int32_t* owners, int64_t n,
                                      float* out);

/* Parameter / optimiser state access (device buffers of n_params floats,
   packed layout).  what: 0 = Theta, 1 = Adam m, 2 = Adam v, 3 = last gradient. */
pinn_dd_status pinn_dd_get_params(pinn_dd* h, int32_t sub, int32_t what, float* dst_dev);
pinn_dd_status pinn_dd_set_params(pinn_dd* h, int32_t sub, int32_t what, const float* src_dev);
/* Adam step counter t of subdomain `sub` (host; synchronises). */
pinn_dd_status pinn_dd_get_step(pinn_dd* h, int32_t sub, int32_t* t);

/* With PINN_DD_FLAG_TIMING: cumulative device milliseconds since the last call
   (synchronises, then resets) of ms8 = {K2 payload, K1 loss+grad, K5
   reduce/adam, launches counted, exchange (NCCL group on the exchange stream,
   from the end of K2), K1 interior part, K1 interface part, exposed exchange
   (time the step's stream waited for the exchange after K1 interior)}.  When
   pinn_dd_step runs fused (below) K2's work is inside K1 and its entry is 0;
   entries 4-7 are 0 without remote twins. */
pinn_dd_status pinn_dd_kernel_times(pinn_dd* h, double* ms8);

/* 1 if pinn_dd_step runs the interface payload (K2) and the loss + gradient
   (K1) as one persistent launch: payload chunks first, interface loss chunks
   wait on a device counter of finished payload chunks (Algorithm 1 lines
   238-262, with every neighbour on this GPU: n_recv == 0).
   0 otherwise (point-per-thread kernel, remote twins, or no interface). */
int32_t pinn_dd_step_fused(const pinn_dd* h);

/* Tile geometry chosen for this handle: {points per tile P, tiles per chunk,
   number of chunks, grid size}. */
pinn_dd_status pinn_dd_plan_info(pinn_dd* h, int64_t* info4);

/* Debug / test access to internal device buffers (library-owned, read-only
   for the caller): 0 point class word, 1 1/N per point, 2 twin row, 3 K1
   chunks, 4 K2 chunks, 5 gradient partials, 6 internal (padded) parameters. */
pinn_dd_status pinn_dd_debug_buffer(pinn_dd* h, int32_t which, void** ptr, int64_t* bytes);

void pinn_dd_destroy(pinn_dd* h);

/* Message of the last failing call on h (NULL h: the last pinn_dd_create /
   workspace_size failure of this thread).  Never NULL. */
const char* pinn_dd_last_error(const pinn_dd* h);

#ifdef __cplusplus
}
#endif
#endif /* PINN_DD_H */
