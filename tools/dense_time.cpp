// Host timing of the Krylov-Schur dense kernels on a random n x n matrix
// (development aid): complex Schur, eigenvectors, reorder, real basis, the
// restart products. Build: g++ -O3 -march=x86-64-v3 -fcx-limited-range -fopenmp
//   -I paper_2112_14064_b200/csrc/host -I paper_2112_14064_b200/csrc tools/dense_time.cpp
#include "dense.cpp"
#include <chrono>
#include <cstdio>
#include <random>
using namespace rqb;
static double ms(std::chrono::steady_clock::time_point a){return std::chrono::duration<double,std::milli>(std::chrono::steady_clock::now()-a).count();}
int main(int argc,char**argv){
  int n = argc>1?atoi(argv[1]):201, p0 = argc>2?atoi(argv[2]):170;
  std::mt19937_64 g(1); std::normal_distribution<double> d;
  std::vector<double> A(n*n); for(auto&x:A) x=d(g);
  for(int rep=0;rep<4;++rep){
    auto t0=std::chrono::steady_clock::now();
    CMat T,Z; complex_schur(A,n,T,Z); double ts=ms(t0);
    t0=std::chrono::steady_clock::now(); CMat Y=triangular_eigvecs(T); double te=ms(t0);
    std::vector<int> idx(n); for(int i=0;i<n;++i) idx[i]=i;
    if (getenv("SHUF")) std::shuffle(idx.begin(), idx.end(), g); else std::sort(idx.begin(),idx.end(),[&](int a,int b){return std::abs(T(a,a))>std::abs(T(b,b));});
    std::vector<int> sel(n,0); for(int i=0;i<p0;++i) sel[idx[i]]=1;
    for(int i=0;i<n;++i) if(sel[i]) for(int q=0;q<n;++q) if(!sel[q] && std::abs(T(q,q)-std::conj(T(i,i)))<1e-10*std::abs(T(i,i))) sel[q]=1;
    int p=0; for(int s:sel) p+=s;
    t0=std::chrono::steady_clock::now();
    std::vector<int> sel0 = sel;
    CMat Tr=T,Zr=Z; schur_reorder(Tr,Zr,sel); double tr=ms(t0); t0=std::chrono::steady_clock::now();
    std::vector<double> Qp; real_basis(Zr,p,Qp); double tb=ms(t0); t0=std::chrono::steady_clock::now();
    int mm=n; const std::vector<double>& Hm=A;
    std::vector<double> HQ(static_cast<size_t>(mm) * p, 0.0), Tp(static_cast<size_t>(p) * p, 0.0);
#pragma omp parallel for schedule(static) num_threads(host_threads()) if (static_cast<int64_t>(mm) * mm * p > 1000000)
    for (int c = 0; c < p; ++c) {
      double* hq = HQ.data() + static_cast<size_t>(c) * mm;
      for (int t = 0; t < mm; ++t) {
        const double q = Qp[t + static_cast<size_t>(c) * mm];
        if (q == 0.0) continue;
        const double* ht = Hm.data() + static_cast<size_t>(t) * mm;
        for (int i = 0; i < mm; ++i) hq[i] += ht[i] * q;
      }
    }
#pragma omp parallel for schedule(static) num_threads(host_threads()) if (static_cast<int64_t>(mm) * p * p > 1000000)
    for (int c = 0; c < p; ++c) {
      const double* hq = HQ.data() + static_cast<size_t>(c) * mm;
      for (int i = 0; i < p; ++i) {
        const double* qi = Qp.data() + static_cast<size_t>(i) * mm;
        double s = 0;
        for (int t = 0; t < mm; ++t) s += qi[t] * hq[t];
        Tp[i + static_cast<size_t>(c) * p] = s;
      }
    }
    double dmax=0;
#pragma omp parallel for schedule(static) reduction(max : dmax) num_threads(host_threads()) if (static_cast<int64_t>(mm) * p * p > 1000000)
      for (int c = 0; c < p; ++c) {
        std::vector<double> rc(HQ.begin() + static_cast<size_t>(c) * mm, HQ.begin() + static_cast<size_t>(c + 1) * mm);
        for (int t = 0; t < p; ++t) {
          const double tc = Tp[t + static_cast<size_t>(c) * p];
          const double* qt = Qp.data() + static_cast<size_t>(t) * mm;
          for (int i = 0; i < mm; ++i) rc[i] -= tc * qt[i];
        }
        for (int i = 0; i < mm; ++i) dmax = std::max(dmax, std::fabs(rc[i]));
      }
    double tp=ms(t0);
    std::vector<double> Tre, Zre; real_schur(A, n, Tre, Zre);
    std::vector<int> s3 = sel0;
    t0=std::chrono::steady_clock::now();
    const int pr = real_schur_reorder(Tre, Zre, n, s3); double trr=ms(t0);
    printf("real reorder p %d: %.2f ms\n", pr, trr);
    printf("n %d p %d threads %d: schur %.2f eigvecs %.2f reorder %.2f real_basis %.2f products %.2f  defect %.1e\n",n,p,host_threads(),ts,te,tr,tb,tp,dmax);
  }
}
