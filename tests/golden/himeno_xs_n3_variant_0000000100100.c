static float p[33][33][65];
#pragma acc declare create(p[0:33][0:33][0:65])
static float bnd[33][33][65];
#pragma acc declare create(bnd[0:33][0:33][0:65])
static float wrk1[33][33][65];
#pragma acc declare create(wrk1[0:33][0:33][0:65])
static float wrk2[33][33][65];
#pragma acc declare create(wrk2[0:33][0:33][0:65])
static float a[4][33][33][65];
#pragma acc declare create(a[0:4][0:33][0:33][0:65])
static float b[3][33][33][65];
#pragma acc declare create(b[0:3][0:33][0:33][0:65])
static float c[3][33][33][65];
#pragma acc declare create(c[0:3][0:33][0:33][0:65])
static int imax, jmax, kmax;
#pragma acc declare create(imax)
#pragma acc declare create(jmax)
#pragma acc declare create(kmax)
static float omega;
#pragma acc declare create(omega)

void initmt()
{
  int i, j, k;
  for(i=0;i<33;i++)
    for(j=0;j<33;j++)
      for(k=0;k<65;k++){
        a[0][i][j][k]=0.0;
        a[1][i][j][k]=0.0;
        a[2][i][j][k]=0.0;
        a[3][i][j][k]=0.0;
        b[0][i][j][k]=0.0;
        b[1][i][j][k]=0.0;
        b[2][i][j][k]=0.0;
        c[0][i][j][k]=0.0;
        c[1][i][j][k]=0.0;
        c[2][i][j][k]=0.0;
        p[i][j][k]=0.0;
        wrk1[i][j][k]=0.0;
        bnd[i][j][k]=0.0;
      }
  for(i=0;i<imax;i++)
    for(j=0;j<jmax;j++)
      for(k=0;k<kmax;k++){
        a[0][i][j][k]=1.0;
        a[1][i][j][k]=1.0;
        a[2][i][j][k]=1.0;
        a[3][i][j][k]=1.0/6.0;
        b[0][i][j][k]=0.0;
        b[1][i][j][k]=0.0;
        b[2][i][j][k]=0.0;
        c[0][i][j][k]=1.0;
        c[1][i][j][k]=1.0;
        c[2][i][j][k]=1.0;
        p[i][j][k]=(float)(i*i)/(float)((imax-1)*(imax-1));
        wrk1[i][j][k]=0.0;
        bnd[i][j][k]=1.0;
      }
}

float jacobi(int nn)
{
  int i, j, k, n;
  float gosa, s0, ss;
  #pragma acc update device(a[0:4][0:33][0:33][0:65])
  #pragma acc update device(b[0:3][0:33][0:33][0:65])
  #pragma acc update device(bnd[0:33][0:33][0:65])
  #pragma acc update device(c[0:3][0:33][0:33][0:65])
  #pragma acc update device(imax)
  #pragma acc update device(jmax)
  #pragma acc update device(kmax)
  #pragma acc update device(omega)
  #pragma acc update device(p[0:33][0:33][0:65])
  #pragma acc update device(wrk1[0:33][0:33][0:65])
  #pragma acc update device(wrk2[0:33][0:33][0:65])
  #pragma acc data copyin(s0,ss)
  for(n=0;n<nn;++n){
    gosa = 0.0;
    #pragma acc data copy(gosa)
    #pragma acc data present(a[0:4][0:33][0:33][0:65],b[0:3][0:33][0:33][0:65],bnd[0:33][0:33][0:65],c[0:3][0:33][0:33][0:65],imax,jmax,kmax,omega,p[0:33][0:33][0:65],s0,ss,wrk1[0:33][0:33][0:65])
    #pragma acc kernels
    for(i=1;i<imax-1;i++)
      for(j=1;j<jmax-1;j++)
        for(k=1;k<kmax-1;k++){
          s0 = a[0][i][j][k] * p[i+1][j][k]
             + a[1][i][j][k] * p[i][j+1][k]
             + a[2][i][j][k] * p[i][j][k+1]
             + b[0][i][j][k] * ( p[i+1][j+1][k] - p[i+1][j-1][k]
                               - p[i-1][j+1][k] + p[i-1][j-1][k] )
             + b[1][i][j][k] * ( p[i][j+1][k+1] - p[i][j-1][k+1]
                               - p[i][j+1][k-1] + p[i][j-1][k-1] )
             + b[2][i][j][k] * ( p[i+1][j][k+1] - p[i-1][j][k+1]
                               - p[i+1][j][k-1] + p[i-1][j][k-1] )
             + c[0][i][j][k] * p[i-1][j][k]
             + c[1][i][j][k] * p[i][j-1][k]
             + c[2][i][j][k] * p[i][j][k-1]
             + wrk1[i][j][k];
          ss = ( s0 * a[3][i][j][k] - p[i][j][k] ) * bnd[i][j][k];
          gosa += ss*ss;
          wrk2[i][j][k] = p[i][j][k] + omega * ss;
        }
    #pragma acc data present(imax,jmax,kmax,p[0:33][0:33][0:65],wrk2[0:33][0:33][0:65])
    #pragma acc kernels
    for(i=1;i<imax-1;++i)
      for(j=1;j<jmax-1;++j)
        for(k=1;k<kmax-1;++k)
          p[i][j][k] = wrk2[i][j][k];
  }
  #pragma acc update self(p[0:33][0:33][0:65])
  return gosa;
}

int main()
{
  float gosa;
  imax = 33-1;
  jmax = 33-1;
  kmax = 65-1;
  omega = 0.8;
  initmt();
  gosa = jacobi(3);
  printf("%.9e\n", gosa);
  printf("%.9e\n", p[16][16][32]);
  printf("%.9e\n", p[1][1][1]);
  printf("%.9e\n", p[30][30][62]);
  printf("%.9e\n", p[11][22][16]);
  return 0;
}
